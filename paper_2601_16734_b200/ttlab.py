"""Python mirror of the reference's hot-path API, executed on the B200.

Names, argument meaning and error behaviour follow `ttlab`
(/root/reference/proj/include/ttlab/): `Strategy` (types.hpp:50-94),
`apply` (blas.hpp:8-11), `hadamard` (blas.hpp:45-67), `simplify`
(simplify.hpp:182-195), `canonicalize` (mps.hpp:310-313), `scprod`
(mps.hpp:416-423), `detail::apply_raw` (mpo.hpp:213-238), `MPSSum` /
`combine` / `simplify(MPSSum)` (mps.hpp:326-405, simplify.hpp:151-215) and
`MPOList` with `apply(MPOList, ...)` (mpo.hpp:109-129, blas.hpp:13-42).  Every operation
runs through the C ABI of `libttgpu.so`; there is no CPU path.

States are `DeviceMPS` handles (device resident, optionally a batch of
identically shaped chains).  Host tensors are lists of numpy arrays shaped
(left, phys, right) for an MPS and (left, out, in, right) for an MPO.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib

UNBOUNDED_BOND = (1 << 63) - 1
SVD_TRUNCATE, VARIATIONAL = 0, 1


class ShapeError(ValueError):
    """shape_error (types.hpp:22-25)."""


class CapacityError(RuntimeError):
    """capacity_error (types.hpp:28-31)."""


class NumericError(RuntimeError):
    """numeric_error (types.hpp:34-37)."""


class DeviceError(RuntimeError):
    """CUDA failure or no B200 visible."""


@dataclass(frozen=True)
class Strategy:
    """types.hpp:50-88."""

    method: int = VARIATIONAL
    tolerance: float = 1e-12
    simplification_tolerance: float = 1e-12
    max_bond: int = UNBOUNDED_BOND
    max_sweeps: int = 4
    normalize: bool = False

    def with_method(self, m):
        return replace(self, method=m)

    def with_tolerance(self, t):
        return replace(self, tolerance=t)

    def with_simplification_tolerance(self, t):
        return replace(self, simplification_tolerance=t)

    def with_max_bond(self, chi):
        return replace(self, max_bond=chi)

    def with_max_sweeps(self, s):
        return replace(self, max_sweeps=s)

    def with_normalize(self, f):
        return replace(self, normalize=f)

    def _c(self) -> _lib.ttg_strategy:
        mb = self.max_bond if self.max_bond < (1 << 31) - 1 else 0
        return _lib.ttg_strategy(int(self.method), float(self.tolerance), float(self.simplification_tolerance),
                                 int(mb), int(self.max_sweeps), int(bool(self.normalize)))


DEFAULT_STRATEGY = Strategy()
NO_TRUNCATION = Strategy(SVD_TRUNCATE, 0.0, 0.0, UNBOUNDED_BOND, 4, False)

_ERRORS = {
    _lib.TTG_SHAPE: ShapeError,
    _lib.TTG_CAPACITY: CapacityError,
    _lib.TTG_NUMERIC: NumericError,
    _lib.TTG_CUDA: DeviceError,
    _lib.TTG_INVALID: ValueError,
}


class Context:
    """One ttg_ctx (CUDA stream + launch counter) per host thread and device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = lib.ttg_create(int(device), C.byref(h))
        if st != _lib.TTG_OK:
            raise DeviceError(f"ttg_create(device={device}) failed with status {st}: no usable CUDA device")
        self.handle = h
        self.device = device
        # device objects allocated on this context's stream: freed before the
        # stream goes away even when the garbage collector finalises the
        # context first (reference cycles at interpreter exit)
        self._live = {}

    def _track(self, handle: C.c_void_p, free):
        self._live[handle.value] = free

    def _release(self, handle: C.c_void_p):
        free = self._live.pop(handle.value, None) if handle and self._live is not None else None
        if free is not None:
            free(handle)

    def check(self, status: int):
        if status != _lib.TTG_OK:
            msg = lib.ttg_last_error(self.handle).decode()
            raise _ERRORS.get(status, RuntimeError)(msg)

    def set_stream(self, stream_ptr: int):
        self.check(lib.ttg_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def synchronize(self):
        self.check(lib.ttg_synchronize(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(lib.ttg_kernel_launches(self.handle))

    # ---- NCCL communicator owned by the context (batched configs) ----
    COMM_ID_BYTES = 128

    def comm_unique_id(self) -> bytes:
        """Rank 0: a fresh communicator id to ship to every rank (ncclGetUniqueId)."""
        buf = C.create_string_buffer(self.COMM_ID_BYTES)
        self.check(lib.ttg_comm_unique_id(self.handle, buf))
        return buf.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Collective over all ranks: the context joins the communicator `uid` (ncclCommInitRank)."""
        if len(uid) != self.COMM_ID_BYTES:
            raise ShapeError("comm_init: the id must be COMM_ID_BYTES long")
        self.check(lib.ttg_comm_init(self.handle, int(nranks), int(rank), C.create_string_buffer(uid, len(uid))))

    def comm_info(self):
        n, r = C.c_int(), C.c_int()
        self.check(lib.ttg_comm_info(self.handle, C.byref(n), C.byref(r)))
        return n.value, r.value

    def allgather_f64(self, send: np.ndarray) -> np.ndarray:
        """send[count] of every rank -> (nranks, count) in rank order (ncclAllGather on the context stream)."""
        send = np.ascontiguousarray(send, dtype=np.float64).ravel()
        n, _ = self.comm_info()
        recv = np.empty((n, send.size), dtype=np.float64)
        self.check(lib.ttg_comm_allgather_f64(self.handle, C.c_void_p(send.ctypes.data), send.size,
                                              C.c_void_p(recv.ctypes.data)))
        return recv

    def comm_free(self):
        self.check(lib.ttg_comm_free(self.handle))

    PROFILE_CLASSES = {"gemm": 0, "svd": 1, "qr": 2, "expand": 3}

    def profile_enable(self, on: bool = True):
        self.check(lib.ttg_profile_enable(self.handle, int(bool(on))))

    def profile_read(self) -> dict:
        out = {}
        for name, cls in self.PROFILE_CLASSES.items():
            n, ms, fl = C.c_int64(), C.c_double(), C.c_double()
            self.check(lib.ttg_profile_read(self.handle, cls, C.byref(n), C.byref(ms), C.byref(fl)))
            out[name] = dict(launches=n.value, ms=ms.value, flops=fl.value)
        sw = C.c_int64()
        self.check(lib.ttg_profile_svd_sweeps(self.handle, C.byref(sw)))
        out["svd"]["jacobi_sweeps"] = sw.value
        return out

    def __del__(self):
        try:
            live, self._live = self._live, None
            for hv, free in (live or {}).items():
                free(C.c_void_p(hv))
            if self.handle:
                lib.ttg_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_tls = threading.local()


def context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _dtype_code(arrs) -> int:
    return _lib.TTG_C128 if any(np.iscomplexobj(a) for a in arrs) else _lib.TTG_F64


def _np_dtype(code):
    return np.complex128 if code == _lib.TTG_C128 else np.float64


def _i64(vals):
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])


class DeviceMPS:
    """Device-resident MPS batch (`ttg_dmps`): `count` chains of one length."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        ctx._track(handle, lib.ttg_mps_free)

    # ---- construction
    @classmethod
    def from_tensors(cls, tensors: Sequence[np.ndarray], error: float = 0.0, ctx: Optional[Context] = None):
        return cls.from_batch([tensors], [error], ctx)

    @classmethod
    def from_batch(cls, chains: Sequence[Sequence[np.ndarray]], errors=None, ctx: Optional[Context] = None):
        ctx = ctx or context()
        code = _dtype_code([t for ch in chains for t in ch])
        dt = _np_dtype(code)
        views = (_lib.ttg_mps_view * len(chains))()
        keep = []
        for i, ch in enumerate(chains):
            arrs = [np.ascontiguousarray(t, dtype=dt) for t in ch]
            for a in arrs:
                if a.ndim != 3:
                    raise ShapeError("MPS tensors must be rank 3 (left, phys, right)")
            for a, b in zip(arrs[:-1], arrs[1:]):
                if a.shape[2] != b.shape[0]:
                    raise ShapeError("MPS bond mismatch between neighboring tensors")
            bonds = _i64([arrs[0].shape[0]] + [a.shape[2] for a in arrs])
            phys = _i64([a.shape[1] for a in arrs])
            ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
            keep += [arrs, bonds, phys, ptrs]
            err = 0.0 if errors is None else float(errors[i])
            views[i] = _lib.ttg_mps_view(len(arrs), code, bonds, phys, ptrs, err)
        h = C.c_void_p()
        ctx.check(lib.ttg_mps_upload(ctx.handle, views, len(chains), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_device(cls, n, dtype_code, count, bonds, phys, dev_ptrs, errors=None, ctx: Optional[Context] = None):
        """Copy device-resident packed site buffers (e.g. torch tensors' data_ptr)."""
        ctx = ctx or context()
        h = C.c_void_p()
        errs = None if errors is None else (C.c_double * count)(*errors)
        ptrs = (C.c_void_p * n)(*dev_ptrs)
        ctx.check(lib.ttg_mps_from_device(ctx.handle, n, dtype_code, count, _i64(bonds), _i64(phys), ptrs, errs,
                                          C.byref(h)))
        return cls(h, ctx)

    def __del__(self):
        try:
            if self.handle:
                self.ctx._release(self.handle)
                self.handle = None
        except Exception:
            pass

    # ---- shape / readback
    def info(self, chain: int = 0):
        n, dt, cnt, ctr = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        err = C.c_double()
        st = lib.ttg_mps_info(self.handle, chain, C.byref(n), C.byref(dt), C.byref(cnt), None, None, None, None)
        if st != _lib.TTG_OK:
            raise ValueError("bad chain index")
        bonds = (C.c_int64 * (n.value + 1))()
        phys = (C.c_int64 * n.value)()
        lib.ttg_mps_info(self.handle, chain, None, None, None, bonds, phys, C.byref(err), C.byref(ctr))
        return dict(n=n.value, dtype=dt.value, count=cnt.value, bonds=list(bonds), phys=list(phys),
                    error=err.value, center=ctr.value)

    def __len__(self):
        return self.info()["n"]

    @property
    def count(self) -> int:
        return self.info()["count"]

    def bond_dimensions(self, chain: int = 0) -> List[int]:
        return self.info(chain)["bonds"]

    def max_bond_dimension(self, chain: int = 0) -> int:
        return max(self.bond_dimensions(chain))

    def error(self, chain: int = 0) -> float:
        return self.info(chain)["error"]

    @property
    def center(self) -> int:
        return self.info()["center"]

    def to_tensors(self, chain: int = 0) -> List[np.ndarray]:
        inf = self.info(chain)
        dt = _np_dtype(inf["dtype"])
        b, p = inf["bonds"], inf["phys"]
        arrs = [np.empty((b[k], p[k], b[k + 1]), dtype=dt) for k in range(inf["n"])]
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        self.ctx.check(lib.ttg_mps_download(self.ctx.handle, self.handle, chain, ptrs))
        return arrs

    def to_tensors_batch(self) -> List[List[np.ndarray]]:
        """Every chain of the batch (ttg_mps_download_batch: pinned staging, one copy per chunk)."""
        first = self.info(0)
        dt = _np_dtype(first["dtype"])
        out, ptrs = [], []
        for c in range(first["count"]):
            inf = first if c == 0 else self.info(c)
            b, p = inf["bonds"], inf["phys"]
            arrs = [np.empty((b[k], p[k], b[k + 1]), dtype=dt) for k in range(inf["n"])]
            out.append(arrs)
            ptrs += [a.ctypes.data for a in arrs]
        self.ctx.check(lib.ttg_mps_download_batch(self.ctx.handle, self.handle, (C.c_void_p * len(ptrs))(*ptrs)))
        return out

    def site_ptr(self, chain: int, k: int):
        ptr, n = C.c_void_p(), C.c_int64()
        if lib.ttg_mps_site_ptr(self.handle, chain, k, C.byref(ptr), C.byref(n)) != _lib.TTG_OK:
            raise ValueError("bad site")
        return ptr.value, n.value


class DeviceMPO:
    """Device-resident MPO (`ttg_dmpo`)."""

    def __init__(self, tensors: Sequence[np.ndarray], ctx: Optional[Context] = None):
        ctx = ctx or context()
        code = _dtype_code(tensors)
        arrs = [np.ascontiguousarray(t, dtype=_np_dtype(code)) for t in tensors]
        for a in arrs:
            if a.ndim != 4:
                raise ShapeError("MPO tensors must be rank 4 (left, out, in, right)")
        for a, b in zip(arrs[:-1], arrs[1:]):
            if a.shape[3] != b.shape[0]:
                raise ShapeError("MPO bond mismatch between neighboring tensors")
        bonds = _i64([arrs[0].shape[0]] + [a.shape[3] for a in arrs])
        view = _lib.ttg_mpo_view(len(arrs), code, bonds, _i64([a.shape[1] for a in arrs]),
                                 _i64([a.shape[2] for a in arrs]),
                                 (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs]))
        h = C.c_void_p()
        ctx.check(lib.ttg_mpo_upload(ctx.handle, C.byref(view), C.byref(h)))
        self.handle, self.ctx = h, ctx
        ctx._track(h, lib.ttg_mpo_free)

    @classmethod
    def _wrap(cls, handle: C.c_void_p, ctx: Context) -> "DeviceMPO":
        obj = cls.__new__(cls)
        obj.handle, obj.ctx = handle, ctx
        ctx._track(handle, lib.ttg_mpo_free)
        return obj

    def __del__(self):
        try:
            if self.handle:
                self.ctx._release(self.handle)
                self.handle = None
        except Exception:
            pass


def _as_mps(v, ctx=None) -> DeviceMPS:
    if isinstance(v, DeviceMPS):
        return v
    return DeviceMPS.from_tensors(list(v), ctx=ctx)


def _as_mpo(op, ctx=None) -> DeviceMPO:
    if isinstance(op, DeviceMPO):
        return op
    return DeviceMPO(list(op), ctx=ctx)


def _reports(n):
    return (_lib.ttg_report * n)()


def _report_dicts(reps, n):
    return [dict(sweeps=r.sweeps, converged=bool(r.converged), residual=r.residual, error=r.error, norm=r.norm,
                 target_norm2=r.target_norm2) for r in reps[:n]]


def apply_raw(op, v) -> DeviceMPS:
    """mpo.hpp:213-238."""
    v = _as_mps(v)
    op = _as_mpo(op, v.ctx)
    h = C.c_void_p()
    v.ctx.check(lib.ttg_apply_raw(v.ctx.handle, op.handle, v.handle, C.byref(h)))
    return DeviceMPS(h, v.ctx)


def hadamard(u, v) -> DeviceMPS:
    """blas.hpp:45-67."""
    u = _as_mps(u)
    v = _as_mps(v, u.ctx)
    h = C.c_void_p()
    u.ctx.check(lib.ttg_hadamard(u.ctx.handle, u.handle, v.handle, C.byref(h)))
    return DeviceMPS(h, u.ctx)


class MPSSum:
    """Lazy weighted sum of states with equal physical dimensions (mps.hpp:326-349).

    The states stay device handles; `join()` materialises the block-diagonal
    concatenation on the GPU (mps.hpp:352-405)."""

    def __init__(self, weights, states, ctx: Optional[Context] = None):
        weights = [complex(w) for w in weights]
        states = list(states)
        if not weights or len(weights) != len(states):
            raise ShapeError("MPSSum: weights and states must be non-empty and match")
        ctx = ctx or next((s.ctx for s in states if isinstance(s, DeviceMPS)), None)
        self.states = [_as_mps(s, ctx) for s in states]
        self.weights = weights
        dims = self.states[0].info()["phys"]
        for s in self.states:
            if s.count != 1:
                raise ShapeError("MPSSum: single-chain states only")
            if s.info()["phys"] != dims:
                raise ShapeError("MPSSum: states must share physical dimensions")

    @property
    def ctx(self) -> Context:
        return self.states[0].ctx

    def terms(self) -> int:
        return len(self.states)

    def __len__(self):
        return len(self.states[0])

    def error(self) -> float:
        """mps.hpp:344-349."""
        return float(sum(abs(w) * s.error() for w, s in zip(self.weights, self.states)))

    def _c_args(self):
        n = len(self.weights)
        wr = (C.c_double * n)(*[w.real for w in self.weights])
        wi = (C.c_double * n)(*[w.imag for w in self.weights])
        hs = (C.c_void_p * n)(*[s.handle.value for s in self.states])
        return n, wr, wi, hs

    def join(self) -> DeviceMPS:
        """mps.hpp:352-405 on the device."""
        n, wr, wi, hs = self._c_args()
        h = C.c_void_p()
        self.ctx.check(lib.ttg_mps_join(self.ctx.handle, n, wr, wi, hs, C.byref(h)))
        return DeviceMPS(h, self.ctx)


class MPOList:
    """Product of MPO factors, the last entry applied first (mpo.hpp:109-129)."""

    def __init__(self, factors=()):
        self.factors = list(factors)

    def terms(self) -> int:
        return len(self.factors)

    def __getitem__(self, k):
        return self.factors[k]

    def push_back(self, op):
        self.factors.append(op)

    def concatenated(self, other: "MPOList") -> "MPOList":
        return MPOList(self.factors + other.factors)


def _simplify_sum(target: MPSSum, strategy: Strategy, guess, report) -> DeviceMPS:
    g = None if guess is None else _as_mps(guess, target.ctx)
    n, wr, wi, hs = target._c_args()
    reps = _reports(1)
    h = C.c_void_p()
    target.ctx.check(lib.ttg_simplify_sum(target.ctx.handle, n, wr, wi, hs, C.byref(strategy._c()),
                                          None if g is None else g.handle, C.byref(h), reps))
    if report is not None:
        report.extend(_report_dicts(reps, 1))
    return DeviceMPS(h, target.ctx)


def combine(weights, states, strategy: Strategy = DEFAULT_STRATEGY, report: Optional[list] = None) -> DeviceMPS:
    """simplify.hpp:151-180: closest MPS under `strategy` to sum_l weights[l] states[l]."""
    weights, states = list(weights), list(states)
    if not weights or len(weights) != len(states):
        raise ShapeError("combine: weights and states must be non-empty and match")
    try:
        target = MPSSum(weights, states)
    except ShapeError as e:
        raise ShapeError(str(e).replace("MPSSum", "combine")) from None
    return _simplify_sum(target, strategy, None, report)


def simplify(target, strategy: Strategy = DEFAULT_STRATEGY, guess=None, report: Optional[list] = None) -> DeviceMPS:
    """simplify.hpp:182-195 (also the batched simplify when `target` is a batch);
    simplify.hpp:197-215 when `target` is an `MPSSum`."""
    if isinstance(target, MPSSum):
        return _simplify_sum(target, strategy, guess, report)
    t = _as_mps(target)
    g = None if guess is None else _as_mps(guess, t.ctx)
    cnt = t.count
    reps = _reports(cnt)
    h = C.c_void_p()
    t.ctx.check(lib.ttg_simplify(t.ctx.handle, t.handle, C.byref(strategy._c()), None if g is None else g.handle,
                                 C.byref(h), reps))
    if report is not None:
        report.extend(_report_dicts(reps, cnt))
    return DeviceMPS(h, t.ctx)


def apply(op, v, strategy: Strategy = DEFAULT_STRATEGY, report: Optional[list] = None) -> DeviceMPS:
    """blas.hpp:8-42: MPO or MPOList onto an MPS (or batch) or an MPSSum."""
    if isinstance(op, MPOList):
        if op.terms() == 0:
            raise ShapeError("apply: empty MPO list")
        last = op.terms() - 1
        state = apply(op[last], v, strategy, report if last == 0 else None)
        for k in range(last - 1, -1, -1):  # report: the final (outermost) factor
            state = apply(op[k], state, strategy, report if k == 0 else None)
        return state
    if isinstance(v, MPSSum):
        dop = _as_mpo(op, v.ctx)
        applied = [apply_raw(dop, s) for s in v.states]
        return _simplify_sum(MPSSum(v.weights, applied), strategy, None, report)
    v = _as_mps(v)
    op = _as_mpo(op, v.ctx)
    cnt = v.count
    reps = _reports(cnt)
    h = C.c_void_p()
    v.ctx.check(lib.ttg_apply(v.ctx.handle, op.handle, v.handle, C.byref(strategy._c()), C.byref(h), reps))
    if report is not None:
        report.extend(_report_dicts(reps, cnt))
    return DeviceMPS(h, v.ctx)


def canonicalize(v, center: int = 0, strategy: Strategy = DEFAULT_STRATEGY,
                 report: Optional[list] = None) -> DeviceMPS:
    """mps.hpp:310-313."""
    v = _as_mps(v)
    cnt = v.count
    reps = _reports(cnt)
    h = C.c_void_p()
    v.ctx.check(lib.ttg_canonicalize(v.ctx.handle, v.handle, int(center), C.byref(strategy._c()), C.byref(h), reps))
    if report is not None:
        report.extend(_report_dicts(reps, cnt))
    return DeviceMPS(h, v.ctx)


def recenter(v, target: int, strategy: Strategy = DEFAULT_STRATEGY, center: Optional[int] = None):
    """CanonicalMPS::recenter / move_center_right / move_center_left (mps.hpp:238-279) on the
    device: returns (moved state, err) with err = sqrt(sum of the squared dropped weights).  The
    moved state keeps the input's error ledger (recenter adds err to it, the single moves do not:
    the caller decides).  `center` defaults to the state's own centre (single chains)."""
    v = _as_mps(v)
    c = v.center if center is None else int(center)
    if c < 0:
        raise ShapeError("recenter: state is not in canonical form (give its centre)")
    h, err = C.c_void_p(), C.c_double()
    v.ctx.check(lib.ttg_recenter(v.ctx.handle, v.handle, c, int(target), C.byref(strategy._c()), C.byref(h),
                                 C.byref(err)))
    return DeviceMPS(h, v.ctx), err.value


def schmidt_split(theta, strategy: Strategy, direction: int = 0, ctx: Optional[Context] = None):
    """schmidt_split (schmidt.hpp:72-89) on the device: returns (a, b, error); direction 0 =
    LEFT_TO_RIGHT (a isometric), 1 = RIGHT_TO_LEFT (b isometric)."""
    ctx = ctx or context()
    th = np.ascontiguousarray(theta)
    cplx = np.iscomplexobj(th)
    th = th.astype(np.complex128 if cplx else np.float64)
    m, n = th.shape
    k = min(m, n)
    a = np.empty(m * k, dtype=th.dtype)
    b = np.empty(k * n, dtype=th.dtype)
    r, err = C.c_int64(), C.c_double()
    ctx.check(lib.ttg_schmidt_split(ctx.handle, _lib.TTG_C128 if cplx else _lib.TTG_F64, m, n,
                                    C.c_void_p(th.ctypes.data), int(direction), C.byref(strategy._c()),
                                    C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data), C.byref(r), C.byref(err)))
    r = r.value
    return a[:m * r].reshape(m, r), b[:r * n].reshape(r, n), err.value


def scprod(u, v) -> np.ndarray:
    """mps.hpp:416-423, one value per chain."""
    u = _as_mps(u)
    v = _as_mps(v, u.ctx)
    cnt = u.count
    re, im = (C.c_double * cnt)(), (C.c_double * cnt)()
    u.ctx.check(lib.ttg_scprod(u.ctx.handle, u.handle, v.handle, re, im))
    out = np.array(re[:]) + 1j * np.array(im[:])
    return out


def load_mps(path, real_if_possible: bool = True, ctx: Optional[Context] = None) -> DeviceMPS:
    """serialize.hpp:82-99 / 116-121: a TTLAB1 MPS file straight into device memory."""
    ctx = ctx or context()
    h = C.c_void_p()
    ctx.check(lib.ttg_mps_load(ctx.handle, str(path).encode(), int(bool(real_if_possible)), C.byref(h)))
    return DeviceMPS(h, ctx)


def save_mps(path, state, chain: int = 0) -> None:
    """serialize.hpp:67-80 / 108-113 (one chain of a batch)."""
    state = _as_mps(state)
    state.ctx.check(lib.ttg_mps_save(state.ctx.handle, state.handle, int(chain), str(path).encode()))


def load_mpo(path, real_if_possible: bool = True, ctx: Optional[Context] = None) -> DeviceMPO:
    """serialize.hpp:101-121 (MPO)."""
    ctx = ctx or context()
    h = C.c_void_p()
    ctx.check(lib.ttg_mpo_load(ctx.handle, str(path).encode(), int(bool(real_if_possible)), C.byref(h)))
    return DeviceMPO._wrap(h, ctx)


def save_mpo(path, op) -> None:
    op = _as_mpo(op)
    op.ctx.check(lib.ttg_mpo_save(op.ctx.handle, op.handle, str(path).encode()))


def expectation_mpo(op, u, v=None) -> np.ndarray:
    """blas.hpp:128-138: <u, op v> per chain (v defaults to u)."""
    u = _as_mps(u)
    dv = None if v is None else _as_mps(v, u.ctx)
    dop = _as_mpo(op, u.ctx)
    cnt = u.count
    re, im = (C.c_double * cnt)(), (C.c_double * cnt)()
    u.ctx.check(lib.ttg_expectation_mpo(u.ctx.handle, dop.handle, u.handle, None if dv is None else dv.handle, re, im))
    return np.array(re[:]) + 1j * np.array(im[:])


def apply_effective_two_site(lenv, w1, w2, renv, x, ctx: Optional[Context] = None) -> np.ndarray:
    """eigensolvers.hpp:15-64 (detail::apply_effective_two_site): y = H_eff x for the two-site
    effective operator, on the device (one DMMA GEMM for the left environment, one kernel for both
    MPO sites, D2 DMMA GEMMs for the right environment).  lenv: D0 matrices L[c0] (chiAo x chiA) or an
    array (D0, chiAo, chiA); w1 (D0, d1o, d1, D1); w2 (D1, d2o, d2, D2); renv: D2 matrices R[c2]
    (chiBo x chiB); x of size chiA d1 d2 chiB ordered (a, s1, s2, B).  Returns y ordered
    (a', s1', s2', b')."""
    L = np.asarray(lenv)
    R = np.asarray(renv)
    w1 = np.asarray(w1)
    w2 = np.asarray(w2)
    x = np.asarray(x).reshape(-1)
    if L.ndim != 3 or R.ndim != 3 or w1.ndim != 4 or w2.ndim != 4:
        raise ShapeError("apply_effective_two_site: bad operand ranks")
    D0, d1o, d1, D1 = w1.shape
    D1b, d2o, d2, D2 = w2.shape
    _, chiAo, chiA = L.shape
    _, chiBo, chiB = R.shape
    if L.shape[0] != D0 or R.shape[0] != D2 or D1b != D1:
        raise ShapeError("apply_effective_two_site: bond mismatch")
    if x.size != chiA * d1 * d2 * chiB:  # eigensolvers.hpp:22-23
        raise ShapeError("apply_effective_two_site: bad vector size")
    cplx = any(np.iscomplexobj(a) for a in (L, R, w1, w2, x))
    dt = np.complex128 if cplx else np.float64
    L, R, w1, w2, x = (np.ascontiguousarray(a, dtype=dt) for a in (L, R, w1, w2, x))
    y = np.empty(chiAo * d1o * d2o * chiBo, dtype=dt)
    dims = (C.c_int * 11)(D0, D1, D2, d1o, d1, d2o, d2, chiAo, chiA, chiBo, chiB)
    ctx = ctx or context()
    ctx.check(lib.ttg_apply_effective_two_site(ctx.handle, _lib.TTG_C128 if cplx else _lib.TTG_F64, dims,
                                               *[C.c_void_p(a.ctypes.data) for a in (L, w1, w2, R, x, y)]))
    return y


def expectation_local(v, op, site: int, op2=None, site2: Optional[int] = None) -> np.ndarray:
    """blas.hpp:100-125: <v, O_site v> or the two-point <v, O_site O2_site2 v>
    (not normalised).  The local operators become a bond-1 MPO (identity on
    the other sites) evaluated by `expectation_mpo` on the device."""
    v = _as_mps(v)
    info = v.info()
    L, phys = info["n"], info["phys"]
    if site < 0 or site >= L:
        raise ShapeError("expectation_local: site out of range")
    if (op2 is None) != (site2 is None):
        raise ShapeError("expectation_local: two-point value needs both operator and site")
    if op2 is not None and (site2 < 0 or site2 >= L or site2 == site):
        raise ShapeError("expectation_local: second site out of range")
    ops = {site: op}
    if op2 is not None:
        ops[site2] = op2
    tensors = []
    for n in range(L):
        m = np.asarray(ops.get(n, np.eye(phys[n])))
        if m.shape != (phys[n], phys[n]):
            raise ShapeError("local operator dimension mismatch")
        tensors.append(m.reshape(1, phys[n], phys[n], 1))
    return expectation_mpo(tensors, v)


def norm(v) -> np.ndarray:
    """MPS::norm (mps.hpp:86) per chain."""
    return np.sqrt(np.maximum(0.0, scprod(v, v).real))
