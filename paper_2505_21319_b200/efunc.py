"""Thin ctypes binding of libefunc (include/efunc.h). Argument marshalling only: every step of
the hot path runs in the library's sm_100a kernels. torch supplies device memory and streams.

Loading fails loudly if the shared library is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# EFUNC_LIB_PATH: an alternative in-tree build of the same library (tuning experiments)
LIB_PATH = os.environ.get("EFUNC_LIB_PATH") or os.path.join(_PKG, "lib", "libefunc.so")

NCH = 13
# model families of Table 3: include/efunc.h efunc_variant
VARIANT_COMBINED, VARIANT_GRID, VARIANT_OFFSET = 0, 1, 2
OK, EINVAL, ESTATE, ENONFINITE, ECUDA, ENOMEM = range(6)
LOSS_NONE, LOSS_MSE, LOSS_MSE_EIKONAL = 0, 1, 2
# default decay mask (reading R-10 / SPEC D15): polynomial coefficients c, g of both banks
DEFAULT_DECAY_MASK = (1 << 1) | (0b111 << 2) | (1 << 9) | (0b111 << 10)

EXPORTED = ["efunc_create", "efunc_destroy", "efunc_forward", "efunc_backward", "efunc_forward_backward",
            "efunc_adamw_step",
            "efunc_eval_grad", "efunc_fit_step", "efunc_mean_shift_init", "efunc_get_params",
            "efunc_set_params", "efunc_get_adam_state", "efunc_set_adam_state", "efunc_set_counting",
            "efunc_get_stats", "efunc_check", "efunc_set_timing", "efunc_get_kernel_ms", "efunc_sync", "efunc_last_error",
            "efunc_mesh", "efunc_channels", "efunc_cosine_replicate", "efunc_cosine_combine",
            "efunc_abi_version", "efunc_set_grad_peers"]


class Config(C.Structure):
    _fields_ = [("R", C.c_int32), ("degree", C.c_int32), ("variant", C.c_int32), ("cutoff_T", C.c_float),
                ("deterministic", C.c_int32), ("device", C.c_int32), ("sync_checks", C.c_int32),
                ("fit_graph", C.c_int32), ("n_shapes", C.c_int32), ("reserved", C.c_int32 * 3)]


class Loss(C.Structure):
    _fields_ = [("kind", C.c_int32), ("eikonal_lambda", C.c_float), ("J_global", C.c_int64)]


class AdamWParams(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("decay_mask", C.c_uint32)]


class Stats(C.Structure):
    _fields_ = [("J", C.c_int64), ("items", C.c_int64), ("candidate_pairs", C.c_double),
                ("kept_pairs", C.c_double), ("beta_min", C.c_float), ("nonfinite", C.c_int32),
                ("overflow_items", C.c_int32), ("kept_pairs_offset", C.c_double), ("launches", C.c_int64),
                ("list_builds", C.c_int64), ("list_entries", C.c_int64), ("list_overflow", C.c_int64)]


class EfuncError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"efunc status {status}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libefunc.so (in-tree build). Raises if it is missing: no fallback path exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libefunc.so not built ({path}); run __graft_entry__.build() or "
                          f"python -m paper_2505_21319_b200.build")
    lib = C.CDLL(path)
    P, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    sig = {
        "efunc_create": [C.POINTER(Config), P, C.POINTER(P)],
        "efunc_destroy": [P],
        "efunc_forward": [P, P, P, i64, C.POINTER(Loss), P, P, P, P],
        "efunc_backward": [P, P, P, P, P],
        "efunc_forward_backward": [P, P, P, i64, C.POINTER(Loss), P, P, P, P],
        "efunc_adamw_step": [P, P, C.POINTER(AdamWParams), P],
        "efunc_eval_grad": [P, P, i64, P, P, P],
        "efunc_fit_step": [P, P, P, i64, C.POINTER(Loss), C.POINTER(AdamWParams), P, P, i32, P],
        "efunc_mean_shift_init": [P, P, i64, f32, P],
        "efunc_get_params": [P, P, i32, P],
        "efunc_set_params": [P, P, i32, P],
        "efunc_get_adam_state": [P, P, P, C.POINTER(i64)],
        "efunc_set_adam_state": [P, P, P, i64],
        "efunc_set_counting": [P, i32],
        "efunc_get_stats": [P, C.POINTER(Stats), P],
        "efunc_check": [P, P],
        "efunc_sync": [P],
        "efunc_set_timing": [P, i32],
        "efunc_set_grad_peers": [P, P, i32, P],
        "efunc_get_kernel_ms": [P, P, i32],
        "efunc_mesh": [P, i32, P, P, f32, P, P, P, P, i64, i64, C.POINTER(i64), C.POINTER(i64), P],
        "efunc_cosine_replicate": [P, i64, i32, P, P],
        "efunc_cosine_combine": [P, i64, i32, P, P, P, i64, P, P, P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.efunc_last_error.argtypes = [P]
    lib.efunc_last_error.restype = C.c_char_p
    lib.efunc_abi_version.argtypes = []
    lib.efunc_abi_version.restype = C.c_int32
    lib.efunc_channels.argtypes = [C.c_int32, C.c_int32]
    lib.efunc_channels.restype = C.c_int32
    _lib = lib
    return lib


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _check_dev(t, name, numel, device):
    import torch
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float32 torch tensor")
    if t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name} must live on cuda:{device}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")


def _check_io(t, name, numel, device, host, pinned=False):
    """fit_step inputs: CUDA tensors on the handle's device, or host (CPU) tensors for host_io
    (pinned when the copy is pipelined): float32, contiguous, exactly numel elements."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float32 torch tensor")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
    if host:
        if t.device.type != "cpu":
            raise ValueError(f"{name} must be a host tensor like q")
        if pinned and not t.is_pinned():
            raise ValueError(f"{name} must be pinned host memory for pipelined host I/O")
    elif t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name} must live on cuda:{device}")


@dataclass
class AdamW:
    lr: float = 6e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 1e-2
    decay_mask: int | None = None  # None: the polynomial coefficients of the handle's layout (SPEC D15)

    def c(self, default_mask: int = DEFAULT_DECAY_MASK) -> AdamWParams:
        mask = default_mask if self.decay_mask is None else self.decay_mask
        return AdamWParams(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, mask)


def _coef_mask(variant: int, degree: int) -> int:
    """Weight-decay mask of a layout (reading R-10, SPEC D15): the polynomial coefficients c, g (and H)
    of every bank; scales s and offsets Delta are not decayed."""
    if variant == VARIANT_COMBINED and degree <= 1:
        return DEFAULT_DECAY_MASK
    coef = {0: 1, 1: 4, 2: 10}[degree]
    mask, o = 0, 0
    if variant != VARIANT_OFFSET:
        mask |= ((1 << coef) - 1) << (o + 1)
        o += 1 + coef
    if variant != VARIANT_GRID:
        mask |= ((1 << coef) - 1) << (o + 4)
    return mask


class EFunc:
    """One efunc grid on one CUDA device: O^{+Delta} with degree-1 polynomials (R^3 x 13) by default,
    or another Table 3 family (variant, degree; R^3 x efunc_channels(variant, degree))."""

    def __init__(self, R: int, theta=None, cutoff_T: float = 20.0, device: int = 0,
                 deterministic: bool = False, sync_checks: bool = False, fit_graph: bool = True,
                 n_shapes: int = 1, degree: int = 1, variant: int = VARIANT_COMBINED):
        """n_shapes > 1: S independent grids in one handle (BASELINE config C5); theta, grads and
        the per-query arrays then carry a leading [S] axis and J counts queries per shape."""
        import torch
        self.lib = load_library()
        self.R = int(R)
        self.S = max(1, int(n_shapes))
        self.device = int(device)
        self.nch = int(self.lib.efunc_channels(int(variant), int(degree)))
        if self.nch < 0:
            raise ValueError(f"unsupported (variant, degree) = ({variant}, {degree})")
        self.n_params = self.S * self.R ** 3 * self.nch
        self.decay_mask = _coef_mask(int(variant), int(degree))
        cfg = Config(self.R, int(degree), int(variant), float(cutoff_T), int(deterministic), self.device,
                     int(sync_checks), int(fit_graph), self.S)
        th = None
        if theta is not None:
            if isinstance(theta, torch.Tensor):
                theta = theta.detach().cpu().numpy()
            th = np.ascontiguousarray(np.asarray(theta, dtype=np.float32).reshape(-1))
            if th.size != self.n_params:
                raise ValueError(f"theta must have n_shapes*R^3*{self.nch} elements")
        h = C.c_void_p()
        st = self.lib.efunc_create(C.byref(cfg), None if th is None else th.ctypes.data, C.byref(h))
        if st != OK:
            raise EfuncError(st, self.lib.efunc_last_error(None).decode())
        self.h = h
        self._torch = torch

    # ---------------------------------------------------------------- helpers
    def _stream(self):
        return self._torch.cuda.current_stream(self.device).cuda_stream

    def _ok(self, st):
        if st != OK:
            raise EfuncError(st, self.lib.efunc_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.efunc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _empty(self, *shape):
        if self.S > 1:
            shape = (self.S,) + shape
        return self._torch.empty(*shape, dtype=self._torch.float32, device=f"cuda:{self.device}")

    def _grad_zeros(self):
        shape = (self.R ** 3, self.nch) if self.S == 1 else (self.S, self.R ** 3, self.nch)
        return self._torch.zeros(*shape, dtype=self._torch.float32, device=f"cuda:{self.device}")

    def _J(self, q):
        """queries per shape"""
        return q.numel() // (3 * self.S)

    def _pshape(self):
        return (self.R ** 3, self.nch) if self.S == 1 else (self.S, self.R ** 3, self.nch)

    # ---------------------------------------------------------------- API
    def forward(self, q, o=None, loss: int = LOSS_NONE, eikonal_lambda: float = 0.1, J_global: int = 0,
                want_O: bool = True, want_G: bool = False, want_loss: bool = True):
        """Returns (O, G, loss) — tensors or None."""
        J = self._J(q)
        _check_dev(q, "q", 3 * J * self.S, self.device)
        _check_dev(o, "o", J * self.S, self.device)
        O = self._empty(J) if want_O else None
        G = self._empty(J, 3) if want_G else None
        L = self._empty(1) if (want_loss and loss != LOSS_NONE) else None
        lc = Loss(loss, eikonal_lambda, J_global)
        self._ok(self.lib.efunc_forward(self.h, _ptr(q), _ptr(o), J, C.byref(lc), _ptr(O), _ptr(G), _ptr(L),
                                        self._stream()))
        return O, G, L

    def backward(self, dL_dO=None, dL_dG=None, grad=None):
        if grad is None:
            grad = self._grad_zeros()
        _check_dev(grad, "grad", self.n_params, self.device)
        _check_dev(dL_dO, "dL_dO", None, self.device)
        _check_dev(dL_dG, "dL_dG", None, self.device)
        self._ok(self.lib.efunc_backward(self.h, _ptr(dL_dO), _ptr(dL_dG), _ptr(grad), self._stream()))
        return grad

    def forward_backward(self, q, o, loss: int = LOSS_MSE, eikonal_lambda: float = 0.1, J_global: int = 0,
                         grad=None, want_O: bool = False, want_loss: bool = True):
        """forward + fused loss upstream + backward in one call (the fused fit kernel for MSE).
        Returns (grad, O, loss); grad is accumulated into (+=) when given."""
        J = self._J(q)
        _check_dev(q, "q", 3 * J * self.S, self.device)
        _check_dev(o, "o", J * self.S, self.device)
        if grad is None:
            grad = self._grad_zeros()
        _check_dev(grad, "grad", self.n_params, self.device)
        O = self._empty(J) if want_O else None
        L = self._empty(1) if want_loss else None
        lc = Loss(loss, eikonal_lambda, J_global)
        self._ok(self.lib.efunc_forward_backward(self.h, _ptr(q), _ptr(o), J, C.byref(lc), _ptr(O), _ptr(grad),
                                                 _ptr(L), self._stream()))
        return grad, O, L

    def adamw_step(self, grad, hp: AdamW | None = None):
        hp = hp or AdamW()
        _check_dev(grad, "grad", self.n_params, self.device)
        p = hp.c(self.decay_mask)
        self._ok(self.lib.efunc_adamw_step(self.h, _ptr(grad), C.byref(p), self._stream()))

    def eval_grad(self, q, want_O=True, want_G=True):
        J = self._J(q)
        _check_dev(q, "q", 3 * J * self.S, self.device)
        O = self._empty(J) if want_O else None
        G = self._empty(J, 3) if want_G else None
        self._ok(self.lib.efunc_eval_grad(self.h, _ptr(q), J, _ptr(O), _ptr(G), self._stream()))
        return O, G

    def mesh(self, N: int, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0), iso: float = 0.0,
             want_lattice: bool = False, want_normals: bool = True):
        """NEXT-3: O on the N^3 lattice over [lo, hi], Marching Cubes at
        iso, unit normals G/|G| at the vertices. Returns (verts [V,3], tris [T,3] int32,
        normals [V,3] or None, lattice O [N,N,N] (z, y, x) or None), all on the handle's device."""
        import torch
        if self.S != 1:
            raise ValueError("mesh() needs a single-shape handle")
        lo3 = (C.c_float * 3)(*lo)
        hi3 = (C.c_float * 3)(*hi)
        nv, nt = C.c_int64(0), C.c_int64(0)
        lat = self._empty(N * N * N) if want_lattice else None
        V, T = 16 * N * N, 32 * N * N  # first guess (a surface crosses ~N^2 cells); retried if short
        for _ in range(2):
            verts = self._empty(max(V, 1), 3)
            normals = self._empty(max(V, 1), 3) if want_normals else None
            tris = torch.empty(max(T, 1), 3, dtype=torch.int32, device=f"cuda:{self.device}")
            self._ok(self.lib.efunc_mesh(self.h, int(N), lo3, hi3, float(iso), _ptr(lat), _ptr(verts),
                                         _ptr(normals), _ptr(tris), V, T, C.byref(nv), C.byref(nt), self._stream()))
            if nv.value <= V and nt.value <= T:
                break
            V, T = nv.value, nt.value
        V, T = nv.value, nt.value
        return (verts[:V], tris[:T], None if normals is None else normals[:V],
                None if lat is None else lat.view(N, N, N))

    def fit_step(self, q, o, hp: AdamW | None = None, loss: int = LOSS_MSE, eikonal_lambda: float = 0.1,
                 J_global: int = 0, grad_ws=None, loss_out=None, pipelined: bool = False):
        """forward + loss + backward + AdamW. q/o either CUDA tensors (async, loss_out a device
        tensor) or pinned CPU tensors (host_io: copies inside the call; returns the loss float).
        pipelined=True with pinned CPU tensors: host_io 2 (the copy of the next step overlaps this
        step's compute); returns a ctypes float array filled in by the time sync() returns."""
        hp = hp or AdamW()
        J = self._J(q)
        lc = Loss(loss, eikonal_lambda, J_global)
        p = hp.c(self.decay_mask)
        host = q.device.type == "cpu"
        _check_io(q, "q", 3 * J * self.S, self.device, host, pinned=host and pipelined)
        _check_io(o, "o", J * self.S, self.device, host, pinned=host and pipelined)
        _check_dev(grad_ws, "grad_ws", self.n_params, self.device)
        if not host:
            _check_dev(loss_out, "loss_out", self.S, self.device)
        if host and pipelined:
            lo = (C.c_float * self.S)()
            self._aio_keep = (getattr(self, "_aio_keep", []) + [(lo, q, o)])[-4:]  # alive until reused
            self._ok(self.lib.efunc_fit_step(self.h, q.data_ptr(), o.data_ptr(), J, C.byref(lc), C.byref(p),
                                             _ptr(grad_ws), C.addressof(lo), 2, self._stream()))
            return lo
        if host:
            lo = (C.c_float * self.S)()
            self._ok(self.lib.efunc_fit_step(self.h, q.data_ptr(), o.data_ptr(), J, C.byref(lc), C.byref(p),
                                             _ptr(grad_ws), C.addressof(lo), 1, self._stream()))
            return float(lo[0]) if self.S == 1 else [float(x) for x in lo]
        self._ok(self.lib.efunc_fit_step(self.h, _ptr(q), _ptr(o), J, C.byref(lc), C.byref(p), _ptr(grad_ws),
                                         _ptr(loss_out), 0, self._stream()))
        return loss_out

    def mean_shift_init(self, surf, bandwidth: float = 100.0):
        N = surf.numel() // (3 * self.S)
        _check_dev(surf, "surf", 3 * N * self.S, self.device)
        self._ok(self.lib.efunc_mean_shift_init(self.h, _ptr(surf), N, float(bandwidth), self._stream()))

    def get_params(self) -> np.ndarray:
        out = np.empty(self._pshape(), dtype=np.float32)
        self._ok(self.lib.efunc_get_params(self.h, out.ctypes.data, 0, self._stream()))
        return out

    def set_params(self, theta):
        th = np.ascontiguousarray(np.asarray(theta, dtype=np.float32).reshape(-1))
        if th.size != self.n_params:
            raise ValueError(f"theta must have n_shapes*R^3*{self.nch} elements")
        self._ok(self.lib.efunc_set_params(self.h, th.ctypes.data, 0, self._stream()))

    def get_adam_state(self):
        m = np.empty(self._pshape(), np.float32)
        v = np.empty_like(m)
        step = C.c_int64(0)
        self._ok(self.lib.efunc_get_adam_state(self.h, m.ctypes.data, v.ctypes.data, C.byref(step)))
        return m, v, int(step.value)

    def set_adam_state(self, m=None, v=None, step: int = 0):
        mm = None if m is None else np.ascontiguousarray(np.asarray(m, np.float32).reshape(-1))
        vv = None if v is None else np.ascontiguousarray(np.asarray(v, np.float32).reshape(-1))
        self._ok(self.lib.efunc_set_adam_state(self.h, None if mm is None else mm.ctypes.data,
                                               None if vv is None else vv.ctypes.data, int(step)))

    def set_counting(self, on: bool):
        self._ok(self.lib.efunc_set_counting(self.h, int(on)))

    def sync(self):
        """wait for the pipelined (host_io 2) fit steps"""
        self._ok(self.lib.efunc_sync(self.h))

    def set_grad_peers(self, peer_ptrs, mc_ptr: int = 0):
        """Fuse the data-parallel gradient reduction into the fold: forward_backward / backward add
        their gradient into every rank's copy of a symmetric buffer (peer_ptrs: device addresses of
        all ranks' copies, e.g. torch symmetric memory buffer_ptrs; mc_ptr: its NVLS multicast
        address or 0). The caller zeroes its copy and synchronises the ranks before the call and
        again before reading it. An empty list and mc_ptr = 0 restore the local fold."""
        ptrs = [int(p) for p in peer_ptrs]
        arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs) if ptrs else None
        self._ok(self.lib.efunc_set_grad_peers(self.h, C.cast(arr, C.c_void_p) if arr is not None else None,
                                               len(ptrs), C.c_void_p(int(mc_ptr)) if mc_ptr else None))

    def set_timing(self, slots: int):
        """Record CUDA events around the dominant kernel of each backward/forward_backward call."""
        self._ok(self.lib.efunc_set_timing(self.h, int(slots)))

    def kernel_ms(self, n: int) -> list:
        buf = (C.c_float * n)()
        self._ok(self.lib.efunc_get_kernel_ms(self.h, C.addressof(buf), int(n)))
        return [float(x) for x in buf]

    def stats(self) -> dict:
        s = Stats()
        self._ok(self.lib.efunc_get_stats(self.h, C.byref(s), self._stream()))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def check(self):
        self._ok(self.lib.efunc_check(self.h, self._stream()))


class CosineStack:
    """Cosine-series stack (§4.4, Eq. cosine-series): S(q) = sum_{b<B} w_b(q) O_b(q),
    w_b(q) = cos(b pi x) cos(b pi y) cos(b pi z) (reading R-C), the B bands Config G-6 models
    (variant GRID, degree 1) of one n_shapes = B handle. theta: [B, R^3, 5]."""

    def __init__(self, R: int = 16, B: int = 4, theta=None, cutoff_T: float = 20.0, device: int = 0):
        self.B = int(B)
        self.bands = EFunc(R, theta, cutoff_T=cutoff_T, device=device, n_shapes=self.B, degree=1,
                           variant=VARIANT_GRID)
        self.lib = self.bands.lib
        self.device = self.bands.device

    def _rep(self, q):
        J = q.numel() // 3
        _check_dev(q, "q", 3 * J, self.device)
        qr = self.bands._empty(J, 3)
        self.bands._ok(self.lib.efunc_cosine_replicate(_ptr(q), J, self.B, _ptr(qr), self.bands._stream()))
        return J, qr

    def forward(self, q, o=None, want_G: bool = False, J_global: int = 0):
        """Returns (S [J], GS [J,3] or None, loss or None); with targets o the band upstreams of the
        MSE loss are kept for backward()."""
        J, qr = self._rep(q)
        O, G, _ = self.bands.forward(qr, want_G=want_G, want_loss=False)
        torch = self.bands._torch
        S = torch.empty(J, device=q.device)
        GS = torch.empty(J, 3, device=q.device) if want_G else None
        up = L = None
        if o is not None:
            _check_dev(o, "o", J, self.device)
            up = torch.empty(self.B, J, device=q.device)
            L = torch.empty(1, device=q.device)
        self.bands._ok(self.lib.efunc_cosine_combine(_ptr(q), J, self.B, _ptr(O), _ptr(G), _ptr(o), int(J_global),
                                                     _ptr(S), _ptr(GS), _ptr(up), _ptr(L), self.bands._stream()))
        self._up = up
        return S, GS, L

    def backward(self, grad=None):
        """dL/dtheta of every band [B, R^3, 5] (+= into grad) from the last forward's MSE upstreams."""
        if getattr(self, "_up", None) is None:
            raise RuntimeError("backward() needs a forward() with targets")
        return self.bands.backward(dL_dO=self._up, grad=grad)

    def adamw_step(self, grad, hp: AdamW | None = None):
        self.bands.adamw_step(grad, hp)
