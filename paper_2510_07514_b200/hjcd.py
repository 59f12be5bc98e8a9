"""Thin ctypes binding of libhjcd.so (include/hjcd.h).

Argument marshalling only: every step of the IK path runs in the library's
CUDA kernels.  torch supplies device memory (tensors, the caching allocator
owns the workspace) and the stream.  There is no CPU fallback: if
libhjcd.so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional, Tuple

from . import inputs as _inputs

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HJCD_LIB", os.path.join(_HERE, "libhjcd.so"))   # override: A/B builds
MAX_DOF = 32

STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported", 3: "CUDA error", 4: "workspace", 5: "nomem"}
TARGET_CONVERGED, TARGET_SUCCESS, TARGET_NOT_CONVERGED, TARGET_INVALID = 0, 1, 2, 3

EXPORTS = [
    "hjcd_robot_create", "hjcd_robot_extend", "hjcd_robot_destroy", "hjcd_robot_dof",
    "hjcd_robot_limits", "hjcd_config_default", "hjcd_workspace_size",
    "hjcd_workspace_size_host", "hjcd_solve", "hjcd_solve_timed", "hjcd_solve_host", "hjcd_ccd",
    "hjcd_solve_batch", "hjcd_select_topn", "hjcd_mmd", "hjcd_workspace_size_f64", "hjcd_solve_f64",
    "hjcd_pjik_f64", "hjcd_pose_error_f64", "hjcd_fk", "hjcd_fk_sfu", "hjcd_poccd", "hjcd_poccd_trace",
    "hjcd_select_replicate", "hjcd_pjik", "hjcd_pjik_trace", "hjcd_select_best", "hjcd_status_string", "hjcd_poccd_kernel",
    "hjcd_last_cuda_error", "hjcd_version",
]


class HjcdError(RuntimeError):
    pass


class hjcd_joint(C.Structure):
    _fields_ = [("type", C.c_int32), ("origin_xyz", C.c_double * 3),
                ("origin_quat_wxyz", C.c_double * 4), ("axis", C.c_double * 3),
                ("lo", C.c_double), ("hi", C.c_double)]


class hjcd_config(C.Structure):
    _fields_ = [("M", C.c_int32), ("K", C.c_int32), ("B", C.c_int32),
                ("ccd_iters", C.c_int32), ("lm_iters", C.c_int32),
                ("target_early_exit", C.c_int32), ("ccd_early_exit", C.c_int32),
                ("eps_p_coarse", C.c_float), ("eps_o_coarse", C.c_float),
                ("eps_p_fine", C.c_float), ("eps_o_fine", C.c_float),
                ("gamma", C.c_float), ("delta0", C.c_float), ("delta_rho", C.c_float),
                ("delta_min", C.c_float), ("sigma_ccd", C.c_float), ("sigma_rep", C.c_float),
                ("sigma_lm", C.c_float), ("lambda_", C.c_float), ("d_floor", C.c_float),
                ("R", C.c_float), ("beta", C.c_float), ("A", C.c_int32),
                ("w_p", C.c_float), ("w_o", C.c_float), ("succ_p", C.c_float),
                ("succ_o", C.c_float), ("tau_deg", C.c_float), ("repl_noise_all", C.c_int32),
                ("rng_seed", C.c_uint64), ("target_index_offset", C.c_int64)]


_lib = None


def lib():
    """Load libhjcd.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HjcdError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P, i32, sz = C.c_void_p, C.c_int32, C.c_size_t
        L.hjcd_robot_create.argtypes = [P, i32, P, P, C.POINTER(P)]
        L.hjcd_robot_extend.argtypes = [P, i32, C.POINTER(P)]
        L.hjcd_robot_destroy.argtypes = [P]
        L.hjcd_robot_destroy.restype = None
        L.hjcd_robot_dof.argtypes = [P]
        L.hjcd_robot_limits.argtypes = [P, P, P]
        L.hjcd_config_default.argtypes = [P]
        L.hjcd_config_default.restype = None
        L.hjcd_workspace_size.argtypes = [P, i32, P, C.POINTER(sz)]
        L.hjcd_workspace_size_host.argtypes = [P, i32, P, C.POINTER(sz)]
        L.hjcd_solve.argtypes = [P, P, P, i32, P, P, P, P, P, sz, P]
        L.hjcd_solve_timed.argtypes = [P, P, P, i32, P, P, P, P, P, sz, P, P]
        L.hjcd_solve_host.argtypes = [P, P, P, i32, P, P, P, P, P, sz, P]
        L.hjcd_fk.argtypes = [P, P, i32, P, P, P]
        L.hjcd_fk_sfu.argtypes = [P, P, i32, P, P, P]
        L.hjcd_pose_error_f64.argtypes = [P, P, P, i32, P, P, P]
        L.hjcd_poccd.argtypes = [P, P, P, i32, P, P, P, P, P, P, P]
        L.hjcd_poccd_trace.argtypes = [P, P, P, i32, P, P, P, P, P, P, P, P, P]
        L.hjcd_ccd.argtypes = [P, P, P, i32, P, P, P, P, P]
        L.hjcd_solve_batch.argtypes = [P, P, P, i32, i32, P, P, P, P, P, sz, P]
        L.hjcd_select_topn.argtypes = [P, P, P, i32, P, P, P, i32, P, P, P, P, P]
        L.hjcd_mmd.argtypes = [P, i32, P, i32, i32, i32, P, P, P]
        L.hjcd_workspace_size_f64.argtypes = [P, i32, P, C.POINTER(sz)]
        L.hjcd_solve_f64.argtypes = [P, P, P, i32, P, P, P, P, P, sz, P]
        L.hjcd_pjik_f64.argtypes = [P, P, P, i32, P, P, P, P, P, P, P]
        L.hjcd_select_replicate.argtypes = [P, P, P, P, i32, P, P, P]
        L.hjcd_pjik.argtypes = [P, P, P, i32, P, P, P, P, P, P, P]
        L.hjcd_pjik_trace.argtypes = [P, P, P, i32, P, P, P, P, P, P, P, P, P]
        L.hjcd_select_best.argtypes = [P, P, P, i32, P, P, P, P, P, P, P, P]
        L.hjcd_status_string.restype = C.c_char_p
        L.hjcd_poccd_kernel.argtypes = [P, P]
        L.hjcd_poccd_kernel.restype = C.c_char_p
        L.hjcd_last_cuda_error.restype = C.c_char_p
        L.hjcd_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != 0:
        msg = lib().hjcd_status_string(st).decode()
        if st == 3:
            msg += ": " + lib().hjcd_last_cuda_error().decode()
        raise HjcdError(f"{what}: {msg}")


# ---------------------------------------------------------------- config
def default_config(**over) -> hjcd_config:
    c = hjcd_config()
    lib().hjcd_config_default(C.byref(c))
    for k, v in over.items():
        setattr(c, "lambda_" if k == "lambda" else k, v)
    return c


def config_from_params(p: dict) -> hjcd_config:
    """hjcd_config from a dict using the same keys as the oracle's params."""
    c = default_config()
    for name, _ in hjcd_config._fields_:
        key = "lambda" if name == "lambda_" else name
        if key in p:
            setattr(c, name, p[key])
    return c


# ---------------------------------------------------------------- robot
class Robot:
    """Immutable robot handle (hjcd_robot_create).  `chain` is an
    inputs.Chain joint table."""

    def __init__(self, chain: "_inputs.Chain", _handle=None):
        self.chain = chain
        if _handle is not None:
            self._h = _handle
        else:
            js = (hjcd_joint * len(chain.joints))()
            for i, j in enumerate(chain.joints):
                js[i].type = j.type
                js[i].origin_xyz[:] = list(j.origin_xyz)
                js[i].origin_quat_wxyz[:] = list(j.origin_quat)
                js[i].axis[:] = list(j.axis)
                js[i].lo, js[i].hi = j.lo, j.hi
            ee_xyz = (C.c_double * 3)(*chain.ee_xyz)
            ee_q = (C.c_double * 4)(*chain.ee_quat)
            h = C.c_void_p()
            _check(lib().hjcd_robot_create(js, len(chain.joints), ee_xyz, ee_q, C.byref(h)),
                   "hjcd_robot_create")
            self._h = h
        self.dof = lib().hjcd_robot_dof(self._h)

    @classmethod
    def panda(cls):
        return cls(_inputs.panda())

    @classmethod
    def fetch_like8(cls):
        return cls(_inputs.fetch_like8())

    @classmethod
    def named(cls, name: str):
        return cls(_inputs.robot(name))

    def extend(self, target_dof: int) -> "Robot":
        h = C.c_void_p()
        _check(lib().hjcd_robot_extend(self._h, target_dof, C.byref(h)), "hjcd_robot_extend")
        return Robot(_inputs.extend(self.chain, target_dof), _handle=h)

    def limits(self):
        lo = (C.c_float * self.dof)()
        hi = (C.c_float * self.dof)()
        _check(lib().hjcd_robot_limits(self._h, lo, hi), "hjcd_robot_limits")
        return list(lo), list(hi)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.hjcd_robot_destroy(h)
            self._h = None


# ---------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_f32(t, shape, name):
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise HjcdError(f"{name} must be a contiguous float32 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise HjcdError(f"{name} shape {tuple(t.shape)} != {tuple(shape)}")
    return t


def workspace_size(robot: Robot, T: int, cfg: hjcd_config, host: bool = False) -> int:
    n = C.c_size_t()
    fn = lib().hjcd_workspace_size_host if host else lib().hjcd_workspace_size
    _check(fn(robot.handle, T, C.byref(cfg), C.byref(n)), "hjcd_workspace_size")
    return n.value


class Workspace:
    """Reusable device workspace (torch caching allocator owns the bytes).
    One solve at a time per workspace: the library refuses (HJCD_E_WORKSPACE)
    a solve on another stream while the last one is in flight."""

    def __init__(self):
        self.buf = None
        self.alloc_stream = None

    def get(self, nbytes: int, device, stream=None):
        """The buffer (grown to nbytes), allocated on `stream` (torch stream) and,
        when reused on another stream, recorded on it so the caching allocator
        never hands the bytes out while that stream may still use them."""
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(device)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            with torch.cuda.stream(s):
                self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            self.alloc_stream = s
        elif self.alloc_stream is None or self.alloc_stream.cuda_stream != s.cuda_stream:
            self.buf.record_stream(s)
        return self.buf


# the default workspaces: one per (device, stream), so solves on different
# streams never share stage buffers
_default_ws = {}


def _ws_for(device, nbytes, ws: Optional[Workspace], stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    if ws is None:
        ws = _default_ws.setdefault((str(device), s.cuda_stream), Workspace())
    return ws.get(nbytes, device, s)


def _stream_of(stream, device):
    torch = _torch()
    return stream if stream is not None else torch.cuda.current_stream(device)


# ---------------------------------------------------------------- API
def solve(robot: Robot, targets, cfg: Optional[hjcd_config] = None, out=None,
          workspace: Optional[Workspace] = None, stream=None, events=None):
    """HJCD-IK for targets [T, 7] (cuda f32).  Returns (q [T, dof], pos_err [T],
    ori_err [T], status [T] int32), all on the targets' device; asynchronous.
    events: optional 5 torch.cuda.Event(enable_timing=True), recorded by the
    library at the stage boundaries (hjcd_solve_timed)."""
    torch = _torch()
    cfg = cfg or default_config()
    T = targets.shape[0]
    _dev_f32(targets, (T, 7), "targets")
    dev = targets.device
    if out is None:
        with torch.cuda.stream(_stream_of(stream, dev)):   # results belong to the solve's stream
            out = (torch.empty((T, robot.dof), dtype=torch.float32, device=dev),
                   torch.empty(T, dtype=torch.float32, device=dev),
                   torch.empty(T, dtype=torch.float32, device=dev),
                   torch.empty(T, dtype=torch.int32, device=dev))
    q, pe, oe, st = out
    nbytes = workspace_size(robot, T, cfg)
    ws = _ws_for(dev, nbytes, workspace, _stream_of(stream, dev))
    evp = None
    if events is not None:
        assert len(events) == 5
        for ev in events:
            if not ev.cuda_event:          # torch creates the event lazily on first record
                ev.record()
        evp = (C.c_void_p * 5)(*[ev.cuda_event for ev in events])
    _check(lib().hjcd_solve_timed(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(q), _ptr(pe),
                                  _ptr(oe), _ptr(st), _ptr(ws), ws.numel(), _stream(stream), evp),
           "hjcd_solve")
    return q, pe, oe, st


def solve_batch(robot: Robot, targets, N: int, cfg: Optional[hjcd_config] = None,
                workspace: Optional[Workspace] = None, stream=None):
    """The best N polished solutions per target (hjcd_solve_batch): returns
    (q [T, N, dof], pos_err [T, N], ori_err [T, N], status [T]); entry 0 is
    hjcd_solve's answer."""
    torch = _torch()
    cfg = cfg or default_config()
    T = targets.shape[0]
    _dev_f32(targets, (T, 7), "targets")
    dev = targets.device
    with torch.cuda.stream(_stream_of(stream, dev)):
        q = torch.empty((T, N, robot.dof), dtype=torch.float32, device=dev)
        pe = torch.empty((T, N), dtype=torch.float32, device=dev)
        oe = torch.empty((T, N), dtype=torch.float32, device=dev)
        st = torch.empty(T, dtype=torch.int32, device=dev)
    nbytes = workspace_size(robot, T, cfg)
    ws = _ws_for(dev, nbytes, workspace, _stream_of(stream, dev))
    _check(lib().hjcd_solve_batch(robot.handle, C.byref(cfg), _ptr(targets), T, N, _ptr(q), _ptr(pe), _ptr(oe),
                                  _ptr(st), _ptr(ws), ws.numel(), _stream(stream)), "hjcd_solve_batch")
    return q, pe, oe, st


def solve_f64(robot: Robot, targets, cfg: Optional[hjcd_config] = None, workspace: Optional[Workspace] = None,
              stream=None):
    """HJCD-IK with the fp64 polish (hjcd_solve_f64): fp32 targets [T, 7] ->
    (q [T, dof] f64, pos_err [T] f64, ori_err [T] f64, status [T] int32)."""
    torch = _torch()
    cfg = cfg or default_config()
    T = targets.shape[0]
    _dev_f32(targets, (T, 7), "targets")
    dev = targets.device
    with torch.cuda.stream(_stream_of(stream, dev)):
        q = torch.empty((T, robot.dof), dtype=torch.float64, device=dev)
        pe = torch.empty(T, dtype=torch.float64, device=dev)
        oe = torch.empty(T, dtype=torch.float64, device=dev)
        st = torch.empty(T, dtype=torch.int32, device=dev)
    n = C.c_size_t()
    _check(lib().hjcd_workspace_size_f64(robot.handle, T, C.byref(cfg), C.byref(n)), "hjcd_workspace_size_f64")
    ws = _ws_for(dev, n.value, workspace, _stream_of(stream, dev))
    _check(lib().hjcd_solve_f64(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(q), _ptr(pe), _ptr(oe), _ptr(st),
                                _ptr(ws), ws.numel(), _stream(stream)), "hjcd_solve_f64")
    return q, pe, oe, st


def pjik_f64(robot: Robot, cfg: hjcd_config, targets, seeds, stream=None):
    """Alg. 4 in fp64: fp32 seeds [T, B, n] -> dict theta [T, B, n], ep, eo [T, B]
    (f64), counts [T, B, 4], iters [T, B]."""
    torch = _torch()
    T, n = targets.shape[0], robot.dof
    _dev_f32(targets, (T, 7), "targets")
    _dev_f32(seeds, (T, cfg.B, n), "seeds")
    d = targets.device
    out = dict(theta=torch.empty((T, cfg.B, n), dtype=torch.float64, device=d),
               ep=torch.empty((T, cfg.B), dtype=torch.float64, device=d),
               eo=torch.empty((T, cfg.B), dtype=torch.float64, device=d),
               counts=torch.empty((T, cfg.B, 4), dtype=torch.int32, device=d),
               iters=torch.empty((T, cfg.B), dtype=torch.int32, device=d))
    _check(lib().hjcd_pjik_f64(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds), _ptr(out["theta"]),
                               _ptr(out["ep"]), _ptr(out["eo"]), _ptr(out["counts"]), _ptr(out["iters"]),
                               _stream(stream)), "hjcd_pjik_f64")
    return out


def select_topn(robot: Robot, cfg: hjcd_config, targets, theta, ep, eo, N: int, stream=None):
    """Best N of the B polished seeds: theta [T, B, n], ep/eo [T, B] -> (q [T, N, n],
    pos_err [T, N], ori_err [T, N], idx [T, N])."""
    torch = _torch()
    T, n = targets.shape[0], robot.dof
    _dev_f32(targets, (T, 7), "targets")
    _dev_f32(theta, (T, cfg.B, n), "theta")
    d = targets.device
    q = torch.empty((T, N, n), dtype=torch.float32, device=d)
    pe = torch.empty((T, N), dtype=torch.float32, device=d)
    oe = torch.empty((T, N), dtype=torch.float32, device=d)
    idx = torch.empty((T, N), dtype=torch.int32, device=d)
    _check(lib().hjcd_select_topn(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(theta), _ptr(ep), _ptr(eo), N,
                                  _ptr(q), _ptr(pe), _ptr(oe), _ptr(idx), _stream(stream)), "hjcd_select_topn")
    return q, pe, oe, idx


def mmd(X, Y, stream=None):
    """Per-target MMD^2 (RBF, median-heuristic bandwidth; hjcd_mmd) of X [T, N, d]
    vs Y [T, N2, d] (cuda f32) -> (mmd2 [T], bandwidth [T])."""
    torch = _torch()
    T, N, dim = X.shape
    N2 = Y.shape[1]
    _dev_f32(X, (T, N, dim), "X")
    _dev_f32(Y, (T, N2, dim), "Y")
    m2 = torch.empty(T, dtype=torch.float32, device=X.device)
    bw = torch.empty(T, dtype=torch.float32, device=X.device)
    _check(lib().hjcd_mmd(_ptr(X), N, _ptr(Y), N2, dim, T, _ptr(m2), _ptr(bw), _stream(stream)), "hjcd_mmd")
    return m2, bw


def solve_host(robot: Robot, targets_host, cfg: Optional[hjcd_config] = None, out=None,
               workspace: Optional[Workspace] = None, stream=None, device=None):
    """HJCD-IK with HOST buffers (numpy or CPU tensors, ideally pinned): the C
    ABI copies H2D, solves, copies D2H and synchronises."""
    import numpy as np
    torch = _torch()
    cfg = cfg or default_config()
    tg = targets_host
    if isinstance(tg, np.ndarray):
        tg = torch.from_numpy(np.ascontiguousarray(tg, dtype=np.float32))
    T = tg.shape[0]
    if out is None:
        out = (torch.empty((T, robot.dof), dtype=torch.float32), torch.empty(T, dtype=torch.float32),
               torch.empty(T, dtype=torch.float32), torch.empty(T, dtype=torch.int32))
    q, pe, oe, st = out
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    # the library launches on the CURRENT device: make it `dev` for the call,
    # and default to that device's current stream
    with torch.cuda.device(dev):
        s = _stream_of(stream, dev)
        nbytes = workspace_size(robot, T, cfg, host=True)
        ws = _ws_for(dev, nbytes, workspace, s)
        _check(lib().hjcd_solve_host(robot.handle, C.byref(cfg), _ptr(tg), T, _ptr(q), _ptr(pe),
                                     _ptr(oe), _ptr(st), _ptr(ws), ws.numel(), s.cuda_stream),
               "hjcd_solve_host")
    return q, pe, oe, st


def fk(robot: Robot, q, jac: bool = False, stream=None, sfu: bool = False):
    """Eq. 1 / Eq. 7 on the GPU: q [N, dof] -> pose [N, 7] (and J [N, 6, dof]).
    sfu=True: the PO-CCD kernel's SFU-sincos FK (hjcd_fk_sfu)."""
    torch = _torch()
    N = q.shape[0]
    _dev_f32(q, (N, robot.dof), "q")
    pose = torch.empty((N, 7), dtype=torch.float32, device=q.device)
    J = torch.empty((N, 6, robot.dof), dtype=torch.float32, device=q.device) if jac else None
    fn = lib().hjcd_fk_sfu if sfu else lib().hjcd_fk
    _check(fn(robot.handle, _ptr(q), N, _ptr(pose), _ptr(J), _stream(stream)), "hjcd_fk")
    return (pose, J) if jac else pose


def pose_error_f64(robot: Robot, q, targets, stream=None):
    """fp64 pose errors of fp32 configurations q [N, dof] against targets [N, 7]
    on the fp64 chain (hjcd_pose_error_f64) -> (pos_err [N], ori_err [N]) f64."""
    torch = _torch()
    N = q.shape[0]
    _dev_f32(q, (N, robot.dof), "q")
    _dev_f32(targets, (N, 7), "targets")
    pe = torch.empty(N, dtype=torch.float64, device=q.device)
    oe = torch.empty(N, dtype=torch.float64, device=q.device)
    _check(lib().hjcd_pose_error_f64(robot.handle, _ptr(q), _ptr(targets), N, _ptr(pe), _ptr(oe), _stream(stream)),
           "hjcd_pose_error_f64")
    return pe, oe


def poccd(robot: Robot, cfg: hjcd_config, targets, seeds=None, stream=None):
    """Alg. 3 stage: -> dict theta [T, n, M], cost, ep, eo [T, M], iters [T, M]."""
    torch = _torch()
    T, n, M = targets.shape[0], robot.dof, cfg.M
    _dev_f32(targets, (T, 7), "targets")
    if seeds is not None:
        _dev_f32(seeds, (T, n, M), "seeds")
    d = targets.device
    out = dict(theta=torch.empty((T, n, M), dtype=torch.float32, device=d),
               cost=torch.empty((T, M), dtype=torch.float32, device=d),
               ep=torch.empty((T, M), dtype=torch.float32, device=d),
               eo=torch.empty((T, M), dtype=torch.float32, device=d),
               iters=torch.empty((T, M), dtype=torch.int32, device=d))
    _check(lib().hjcd_poccd(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds),
                            _ptr(out["theta"]), _ptr(out["cost"]), _ptr(out["ep"]),
                            _ptr(out["eo"]), _ptr(out["iters"]), _stream(stream)), "hjcd_poccd")
    return out


def poccd_trace(robot: Robot, cfg: hjcd_config, targets, seeds=None, stream=None, history: bool = False):
    """hjcd_poccd that also returns every seed's decision words:
    trace [T, M, ccd_iters] uint32 (as int32), unwritten past iters = 0, and
    with history=True theta_hist [T, M, ccd_iters + 1, n] (theta at the start
    of every iteration, NaN past iters)."""
    torch = _torch()
    T, n, M = targets.shape[0], robot.dof, cfg.M
    _dev_f32(targets, (T, 7), "targets")
    if seeds is not None:
        _dev_f32(seeds, (T, n, M), "seeds")
    d = targets.device
    out = dict(theta=torch.empty((T, n, M), dtype=torch.float32, device=d),
               cost=torch.empty((T, M), dtype=torch.float32, device=d),
               ep=torch.empty((T, M), dtype=torch.float32, device=d),
               eo=torch.empty((T, M), dtype=torch.float32, device=d),
               iters=torch.empty((T, M), dtype=torch.int32, device=d),
               trace=torch.zeros((T, M, max(cfg.ccd_iters, 1)), dtype=torch.int32, device=d))
    if history:
        out["theta_hist"] = torch.full((T, M, cfg.ccd_iters + 1, n), float("nan"), dtype=torch.float32, device=d)
    _check(lib().hjcd_poccd_trace(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds),
                                  _ptr(out["theta"]), _ptr(out["cost"]), _ptr(out["ep"]), _ptr(out["eo"]),
                                  _ptr(out["iters"]), _ptr(out["trace"]), _ptr(out.get("theta_hist")),
                                  _stream(stream)), "hjcd_poccd_trace")
    return out


def ccd(robot: Robot, cfg: hjcd_config, targets, seeds=None, stream=None):
    """Classic position-only CCD (Alg. 1): -> dict theta [T, n, M], ep [T, M], iters [T, M]."""
    torch = _torch()
    T, n, M = targets.shape[0], robot.dof, cfg.M
    _dev_f32(targets, (T, 7), "targets")
    if seeds is not None:
        _dev_f32(seeds, (T, n, M), "seeds")
    d = targets.device
    out = dict(theta=torch.empty((T, n, M), dtype=torch.float32, device=d),
               ep=torch.empty((T, M), dtype=torch.float32, device=d),
               iters=torch.empty((T, M), dtype=torch.int32, device=d))
    _check(lib().hjcd_ccd(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds), _ptr(out["theta"]),
                          _ptr(out["ep"]), _ptr(out["iters"]), _stream(stream)), "hjcd_ccd")
    return out


def select_replicate(robot: Robot, cfg: hjcd_config, cost, theta, stream=None):
    """Alg. 2 l.2-8: cost [T, M], theta [T, n, M] -> seeds [T, B, n], kept [T, K]."""
    torch = _torch()
    T, n = cost.shape[0], robot.dof
    _dev_f32(cost, (T, cfg.M), "cost")
    _dev_f32(theta, (T, n, cfg.M), "theta")
    seeds = torch.empty((T, cfg.B, n), dtype=torch.float32, device=cost.device)
    kept = torch.empty((T, cfg.K), dtype=torch.int32, device=cost.device)
    _check(lib().hjcd_select_replicate(robot.handle, C.byref(cfg), _ptr(cost), _ptr(theta), T,
                                       _ptr(seeds), _ptr(kept), _stream(stream)),
           "hjcd_select_replicate")
    return seeds, kept


def pjik(robot: Robot, cfg: hjcd_config, targets, seeds, stream=None):
    """Alg. 4 stage: seeds [T, B, n] -> dict theta [T, B, n], ep, eo [T, B],
    counts [T, B, 4], iters [T, B]."""
    torch = _torch()
    T, n = targets.shape[0], robot.dof
    _dev_f32(targets, (T, 7), "targets")
    _dev_f32(seeds, (T, cfg.B, n), "seeds")
    d = targets.device
    # slots >= floor(B/K)*K are not written by the kernel (left uninitialised)
    out = dict(theta=torch.empty((T, cfg.B, n), dtype=torch.float32, device=d),
               ep=torch.empty((T, cfg.B), dtype=torch.float32, device=d),
               eo=torch.empty((T, cfg.B), dtype=torch.float32, device=d),
               counts=torch.empty((T, cfg.B, 4), dtype=torch.int32, device=d),
               iters=torch.empty((T, cfg.B), dtype=torch.int32, device=d))
    _check(lib().hjcd_pjik(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds),
                           _ptr(out["theta"]), _ptr(out["ep"]), _ptr(out["eo"]),
                           _ptr(out["counts"]), _ptr(out["iters"]), _stream(stream)), "hjcd_pjik")
    return out


def pjik_trace(robot: Robot, cfg: hjcd_config, targets, seeds, stream=None, history: bool = False):
    """hjcd_pjik that also returns every seed's decision words:
    trace [T, B, lm_iters] uint32 (as int32), zero where no step was taken, and
    with history=True theta_hist [T, B, lm_iters + 1, n] (theta at the start
    of every iteration, NaN past iters)."""
    torch = _torch()
    T, n = targets.shape[0], robot.dof
    _dev_f32(targets, (T, 7), "targets")
    _dev_f32(seeds, (T, cfg.B, n), "seeds")
    d = targets.device
    out = dict(theta=torch.empty((T, cfg.B, n), dtype=torch.float32, device=d),
               ep=torch.empty((T, cfg.B), dtype=torch.float32, device=d),
               eo=torch.empty((T, cfg.B), dtype=torch.float32, device=d),
               counts=torch.empty((T, cfg.B, 4), dtype=torch.int32, device=d),
               iters=torch.empty((T, cfg.B), dtype=torch.int32, device=d),
               trace=torch.zeros((T, cfg.B, max(cfg.lm_iters, 1)), dtype=torch.int32, device=d))
    if history:
        out["theta_hist"] = torch.full((T, cfg.B, cfg.lm_iters + 1, n), float("nan"), dtype=torch.float32, device=d)
    _check(lib().hjcd_pjik_trace(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(seeds),
                                 _ptr(out["theta"]), _ptr(out["ep"]), _ptr(out["eo"]), _ptr(out["counts"]),
                                 _ptr(out["iters"]), _ptr(out["trace"]), _ptr(out.get("theta_hist")),
                                 _stream(stream)), "hjcd_pjik_trace")
    return out


def select_best(robot: Robot, cfg: hjcd_config, targets, theta, ep_all, eo_all, stream=None):
    torch = _torch()
    T, n = targets.shape[0], robot.dof
    d = targets.device
    q = torch.empty((T, n), dtype=torch.float32, device=d)
    pe = torch.empty(T, dtype=torch.float32, device=d)
    oe = torch.empty(T, dtype=torch.float32, device=d)
    st = torch.empty(T, dtype=torch.int32, device=d)
    _check(lib().hjcd_select_best(robot.handle, C.byref(cfg), _ptr(targets), T, _ptr(theta),
                                  _ptr(ep_all), _ptr(eo_all), _ptr(q), _ptr(pe), _ptr(oe),
                                  _ptr(st), _stream(stream)), "hjcd_select_best")
    return q, pe, oe, st


def poccd_kernel(robot: Robot, cfg: hjcd_config) -> str:
    """Name of the PO-CCD kernel hjcd_solve launches for this robot / config."""
    return lib().hjcd_poccd_kernel(robot.handle, C.byref(cfg)).decode()


def version() -> str:
    return lib().hjcd_version().decode()


def exported_symbols():
    """Names of EXPORTS that the loaded library actually defines."""
    L = lib()
    return [s for s in EXPORTS if hasattr(L, s)]
