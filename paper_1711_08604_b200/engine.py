"""Device-level engine: plans and torch-tensor entry points over the C ABI.

PyTorch is used only for device memory, streams and the host<->device
handoff; every computation is a kernel of libafd_b200.so.  All functions
here take / return CUDA tensors (complex128, row-major ``[batch, N]``), so
callers that keep data resident in HBM never touch the host.

Host tables are built with numpy exactly as the reference builds them
(``transform.py:65`` twiddles, ``core.py:87`` circle, ``transform.py:153``
scales), so the device starts from the reference's bits.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _capi

try:  # torch is plumbing only; the product cannot run without it and a GPU
    import torch
except ImportError as exc:  # pragma: no cover
    raise _capi.AfdCudaUnavailable("torch is required for device memory") from exc

__all__ = ["Plan", "Comm", "get_plan", "host_tables", "DeviceDecomposition", "require_cuda"]


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise _capi.AfdCudaUnavailable(
            "no CUDA device: the B200 engine has no CPU fallback")
    _capi.load()
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)


def host_tables(radii, n):
    """(twiddles, circle, scales) exactly as the reference computes them."""
    r = np.ascontiguousarray(radii, dtype=np.float64)
    tw = np.ascontiguousarray(np.exp(-2j * np.pi * np.arange(n // 2) / n))  # transform.py:65
    circle = np.ascontiguousarray(np.exp(2j * np.pi * np.arange(n) / n))     # core.py:87
    scales = np.ascontiguousarray(np.sqrt(1.0 - r * r) / (n * (1.0 - r ** n)))  # transform.py:153
    return tw, circle, scales


def _locked(fn):
    """Run a Plan method under the plan's lock (the plan's device buffers and
    cached graph are shared by all its entry points).  Work is stream-ordered,
    so a call on a different stream than the previous one first waits for
    the previous call's work (an event recorded after every call)."""
    def wrapper(self, *a, **kw):
        with self.lock:
            st = kw.get("stream") or torch.cuda.current_stream(self.device)
            if self._last_stream is not None and st != self._last_stream:
                st.wait_event(self._done)
            out = fn(self, *a, **kw)
            if self._done is None:
                self._done = torch.cuda.Event()
            self._done.record(st)
            self._last_stream = st
            return out
    wrapper.__name__, wrapper.__doc__ = fn.__name__, fn.__doc__
    return wrapper


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


@dataclass
class DeviceDecomposition:
    steps: torch.Tensor      # uint8 [batch, max_terms, 72] (afd_step records)
    n_steps: torch.Tensor    # int32 [batch]
    initial: torch.Tensor    # float64 [batch]
    remainder: torch.Tensor  # complex128 [batch, N]

    def host_steps(self):
        """(steps structured array [batch, max_terms], n_steps) on the host."""
        raw = self.steps.cpu().numpy()
        return raw.view(_capi.STEP_DTYPE)[..., 0], self.n_steps.cpu().numpy()


class Plan:
    """One afd_plan: device tables for (N, radii, radius shard, batch).

    ``fast=1`` builds an AFD_PLAN_FAST plan (FMA-fused field arithmetic, r^l
    on chip; identical selections, ~1e-14 relative instead of bit-exact);
    ``fast=2`` also tracks each step's top-2 margin (AFD_PLAN_MARGINS).
    A plan's device buffers are shared by all its entry points, so every
    call holds the plan's lock (concurrent callers serialise instead of
    corrupting each other's state)."""

    def __init__(self, radii, n, m0=0, m1=None, max_batch=1, device=None, engine=0, fast=0):
        self.device = require_cuda(device)
        self.lib = _capi.load()
        self.radii = tuple(float(r) for r in radii)
        self.n = int(n)
        self.m = len(self.radii)
        self.m0 = int(m0)
        self.m1 = self.m if m1 is None else int(m1)
        self.max_batch = int(max_batch)
        self.fast = int(fast)
        if self.fast not in (0, 1, 2):
            raise ValueError("fast must be 0, 1 or 2 (with margins), got %r" % (fast,))
        self.lock = threading.RLock()
        self._last_stream, self._done = None, None
        tw, circle, scales = host_tables(self.radii, self.n)
        r = np.ascontiguousarray(self.radii, dtype=np.float64)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _capi.check(self.lib.afd_plan_create(
                C.byref(handle), self.device.index, self.n, self.m, self.m0, self.m1,
                self.max_batch, r.ctypes.data, scales.ctypes.data, tw.ctypes.data,
                circle.ctypes.data, (_capi.PLAN_FAST if self.fast else 0) |
                (_capi.PLAN_MARGINS if self.fast == 2 else 0)))
        self.handle = handle
        self._keep = (tw, circle, scales, r)
        self.engine = int(engine)
        if self.engine:
            _capi.check(self.lib.afd_plan_set_engine(handle, self.engine))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.afd_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self.handle = None

    # -- helpers ------------------------------------------------------------
    def _signal(self, g, batch=None):
        g = g.to(device=self.device, dtype=torch.complex128).contiguous()
        if g.dim() == 1:
            g = g.unsqueeze(0)
        if g.shape[-1] != self.n:
            raise ValueError("signal length %d does not match plan N %d" % (g.shape[-1], self.n))
        if g.shape[0] > self.max_batch:
            raise ValueError("batch %d exceeds plan max_batch %d" % (g.shape[0], self.max_batch))
        return g

    def launch_count(self):
        return int(self.lib.afd_launch_count(self.handle))

    @_locked
    def field_split(self, stream=None):
        """(on-chip rows, two-pass rows) of the last large-N fast field
        evaluation (afd_field_split): the pruned 4096-point transforms vs
        pass A + the column pass."""
        a, b = C.c_int64(), C.c_int64()
        _capi.check(self.lib.afd_field_split(self.handle, C.byref(a), C.byref(b),
                                             _stream(stream)))
        return a.value, b.value

    def field_tiers(self, stream=None):
        """(rows of at most 1024 points, 4096-point rows, two-pass rows) of the last
        large-N fast field evaluation (afd_field_tiers)."""
        out = (C.c_int64 * 3)()
        _capi.check(self.lib.afd_field_tiers(self.handle, out, _stream(stream)))
        return tuple(out)

    def field_tier_rows(self, stream=None):
        """{spectrum terms: rows} of the last large-N fast field evaluation by
        tier, in row order (afd_field_tier_rows): 32, 64, 128 (register
        tiers), 256, 512 (when in use), 1024, 4096 (on-chip transforms), N
        (two-pass; batches of on-chip N: the N-point field kernel, rows
        summed over the signals)."""
        terms, rows, cnt = (C.c_int64 * 8)(), (C.c_int64 * 8)(), C.c_int()
        _capi.check(self.lib.afd_field_tier_rows(self.handle, terms, rows, 8, C.byref(cnt),
                                                 _stream(stream)))
        return {int(terms[t]): int(rows[t]) for t in range(cnt.value)}

    def time_field(self, ghat, reps=20, stream=None):
        """Mean CUDA-event time (ms) of one fused field+argmax launch."""
        ghat = self._signal(ghat)
        ms = C.c_double()
        _capi.check(self.lib.afd_time_field(self.handle, _ptr(ghat), ghat.shape[0], int(reps),
                                            C.byref(ms), _stream(stream)))
        return ms.value

    # -- transforms -----------------------------------------------------------
    @_locked
    def _fft(self, fn, x, stream=None):
        x = self._signal(x)
        out = torch.empty_like(x)
        _capi.check(fn(self.handle, _ptr(x), _ptr(out), x.shape[0], _stream(stream)))
        return out

    def dft_forward(self, x, stream=None):
        return self._fft(self.lib.afd_dft_forward, x, stream)

    def dft_inverse(self, c, stream=None):
        return self._fft(self.lib.afd_dft_inverse, c, stream)

    def analytic_projection(self, x, stream=None):
        return self._fft(self.lib.afd_analytic_projection, x, stream)

    @_locked
    def field(self, ghat, r0=None, r1=None, stream=None):
        ghat = self._signal(ghat)[0]
        r0 = self.m0 if r0 is None else int(r0)
        r1 = self.m1 if r1 is None else int(r1)
        out = torch.empty((max(r1 - r0, 0), self.n), dtype=torch.complex128, device=self.device)
        _capi.check(self.lib.afd_field(self.handle, _ptr(ghat), _ptr(out), r0, r1,
                                       _stream(stream)))
        return out

    @_locked
    def field_direct(self, g, r0=None, r1=None, stream=None):
        """oracle.field_direct rows (direct engine) of one signal g (not its spectrum)."""
        g = self._signal(g)[0]
        r0 = self.m0 if r0 is None else int(r0)
        r1 = self.m1 if r1 is None else int(r1)
        out = torch.empty((max(r1 - r0, 0), self.n), dtype=torch.complex128, device=self.device)
        _capi.check(self.lib.afd_field_direct(self.handle, _ptr(g), _ptr(out), r0, r1,
                                              _stream(stream)))
        return out

    @_locked
    def field_argmax(self, ghat, stream=None):
        ghat = self._signal(ghat)
        out = torch.empty((ghat.shape[0], 32), dtype=torch.uint8, device=self.device)
        _capi.check(self.lib.afd_field_argmax(self.handle, _ptr(ghat), _ptr(out), ghat.shape[0],
                                              _stream(stream)))
        return out

    @_locked
    def argmax(self, field, stream=None):
        field = field.to(device=self.device, dtype=torch.complex128).contiguous()
        if field.dim() != 2 or field.shape[1] != self.n:
            raise ValueError("field must be (rows, N)")
        out = torch.empty(32, dtype=torch.uint8, device=self.device)
        _capi.check(self.lib.afd_argmax(self.handle, _ptr(field), field.shape[0], _ptr(out),
                                        _stream(stream)))
        return out

    @_locked
    def atom(self, kind, a, c=0j, g=None, stream=None, norm=None):
        """Pointwise atom `kind` of afd_atom; `norm` = sqrt(1 - abs(a) ** 2)
        computed by the caller (None: formed on the device)."""
        a = complex(a)
        c = complex(c)
        out = torch.empty(self.n, dtype=torch.complex128, device=self.device)
        if g is not None:
            g = self._signal(g)[0]
        _capi.check(self.lib.afd_atom(self.handle, kind, _ptr(g), a.real, a.imag, c.real, c.imag,
                                      float("nan") if norm is None else float(norm),
                                      _ptr(out), _stream(stream)))
        return out

    @_locked
    def energy(self, g, stream=None):
        g = self._signal(g)
        out = torch.empty(g.shape[0], dtype=torch.float64, device=self.device)
        _capi.check(self.lib.afd_energy(self.handle, _ptr(g), _ptr(out), g.shape[0],
                                        _stream(stream)))
        return out

    @_locked
    def energy_diff(self, g, s, stream=None):
        g = self._signal(g)
        s = self._signal(s)
        out = torch.empty(g.shape[0], dtype=torch.float64, device=self.device)
        _capi.check(self.lib.afd_energy_diff(self.handle, _ptr(g), _ptr(s), _ptr(out),
                                             g.shape[0], _stream(stream)))
        return out

    # -- the hot path -----------------------------------------------------------
    @_locked
    def decompose(self, g, max_terms, threshold=None, dc_first=False, stream=None, out=None):
        """Device-resident decomposition of g ([batch, N] CUDA complex128)."""
        g = self._signal(g)
        b = g.shape[0]
        if out is None:
            out = self.alloc_outputs(b, max_terms)
        _capi.check(self.lib.afd_decompose(
            self.handle, _ptr(g), b, int(max_terms),
            0.0 if threshold is None else float(threshold), int(bool(dc_first)),
            _ptr(out.steps), _ptr(out.n_steps), _ptr(out.initial), _ptr(out.remainder),
            _stream(stream)))
        return out

    @_locked
    def decompose_host(self, signals, max_terms, threshold=None, dc_first=False, stream=None):
        """Host numpy [batch, N] in -> host results out (afd_decompose_host).

        Returns (steps structured [batch, max_terms], n_steps, initial,
        remainder [batch, N], h2d_bytes, d2h_bytes)."""
        sig = np.ascontiguousarray(signals, dtype=np.complex128)
        if sig.ndim == 1:
            sig = sig[None, :]
        b = sig.shape[0]
        steps = np.empty((b, int(max_terms)), dtype=_capi.STEP_DTYPE)
        n_steps = np.empty(b, dtype=np.int32)
        initial = np.empty(b, dtype=np.float64)
        rem = np.empty((b, self.n), dtype=np.complex128)
        h2d, d2h = C.c_int64(), C.c_int64()
        _capi.check(self.lib.afd_decompose_host(
            self.handle, sig.ctypes.data, b, int(max_terms),
            0.0 if threshold is None else float(threshold), int(bool(dc_first)),
            steps.ctypes.data, n_steps.ctypes.data, initial.ctypes.data, rem.ctypes.data,
            C.byref(h2d), C.byref(d2h), _stream(stream)))
        return steps, n_steps, initial, rem, h2d.value, d2h.value

    def alloc_outputs(self, batch, max_terms):
        dev = self.device
        return DeviceDecomposition(
            steps=torch.empty((batch, max_terms, _capi.STEP_DTYPE.itemsize), dtype=torch.uint8,
                              device=dev),
            n_steps=torch.empty(batch, dtype=torch.int32, device=dev),
            initial=torch.empty(batch, dtype=torch.float64, device=dev),
            remainder=torch.empty((batch, self.n), dtype=torch.complex128, device=dev))

    @_locked
    def error_trace(self, g, dec, stream=None, norms=None):
        """errors [batch, max_terms] and reconstructions [batch, N] (device).
        norms: optional [batch, max_terms] float64 tensor of the poles'
        sqrt(1 - abs(a) ** 2) from the caller's scalar arithmetic."""
        g = self._signal(g)
        b, max_terms = dec.steps.shape[0], dec.steps.shape[1]
        errors = torch.zeros((b, max_terms), dtype=torch.float64, device=self.device)
        recon = torch.empty((b, self.n), dtype=torch.complex128, device=self.device)
        if norms is not None:
            norms = norms.to(device=self.device, dtype=torch.float64).contiguous()
        _capi.check(self.lib.afd_error_trace(self.handle, _ptr(g), _ptr(dec.steps), max_terms,
                                             _ptr(dec.n_steps), b, _ptr(norms), _ptr(errors),
                                             _ptr(recon), _stream(stream)))
        return errors, recon

    # -- radius-sharded stepping (multi-GPU) ---------------------------------------
    @_locked
    def decompose_sharded(self, comm, g, max_terms, threshold=None, dc_first=False, stream=None,
                          out=None):
        """Device-resident radius-sharded decomposition over `comm` (a Comm):
        the plan's rows are this rank's shard; one CUDA graph per call shape,
        NCCL all-gathers inside it (afd_decompose_sharded)."""
        g = self._signal(g)
        b = g.shape[0]
        if out is None:
            out = self.alloc_outputs(b, max_terms)
        _capi.check(self.lib.afd_decompose_sharded(
            self.handle, comm.handle, _ptr(g), b, int(max_terms),
            0.0 if threshold is None else float(threshold), int(bool(dc_first)),
            _ptr(out.steps), _ptr(out.n_steps), _ptr(out.initial), _ptr(out.remainder),
            _stream(stream)))
        return out

    @_locked
    def sharded_begin(self, g, stream=None):
        g = self._signal(g)
        _capi.check(self.lib.afd_sharded_begin(self.handle, _ptr(g), g.shape[0], _stream(stream)))
        return g.shape[0]

    @_locked
    def select_local(self, k, dc_first, batch, stream=None):
        out = torch.empty((batch, 32), dtype=torch.uint8, device=self.device)
        _capi.check(self.lib.afd_select_local(self.handle, int(k), int(bool(dc_first)), _ptr(out),
                                              batch, _stream(stream)))
        return out

    @_locked
    def apply_step(self, k, max_terms, threshold, dc_first, cands, steps, stream=None):
        """cands: uint8 [batch, ncand, 32] (rank-major), steps: uint8 [batch, max_terms, 72]."""
        cands = cands.contiguous()
        _capi.check(self.lib.afd_apply_step(
            self.handle, int(k), int(max_terms), 0.0 if threshold is None else float(threshold),
            int(bool(dc_first)), _ptr(cands), cands.shape[1], cands.shape[0], _ptr(steps),
            _stream(stream)))

    @_locked
    def sharded_finish(self, batch, stream=None):
        dev = self.device
        n_steps = torch.empty(batch, dtype=torch.int32, device=dev)
        initial = torch.empty(batch, dtype=torch.float64, device=dev)
        rem = torch.empty((batch, self.n), dtype=torch.complex128, device=dev)
        stopped = torch.empty(batch, dtype=torch.int32, device=dev)
        _capi.check(self.lib.afd_sharded_finish(self.handle, batch, _ptr(n_steps), _ptr(initial),
                                                _ptr(rem), _ptr(stopped), _stream(stream)))
        return n_steps, initial, rem, stopped


class Comm:
    """An afd_comm (NCCL communicator of the library) for `world` ranks."""

    def __init__(self, uid, world, rank, device=None):
        self.device = require_cuda(device)
        self.lib = _capi.load()
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        _capi.check(self.lib.afd_comm_init(C.byref(h), buf, int(world), int(rank),
                                           self.device.index))
        self.handle, self.world, self.rank = h, int(world), int(rank)

    @staticmethod
    def unique_id():
        buf = C.create_string_buffer(128)
        _capi.check(_capi.load().afd_comm_unique_id(buf))
        return buf.raw

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.afd_comm_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self.handle = None


def fp64_peak_tflops(device=None, stream=None):
    """Measured DFMA throughput of this GPU (TFLOP/s, 2 flops per DFMA)."""
    dev = require_cuda(device)
    out = C.c_double()
    _capi.check(_capi.load().afd_fp64_peak(dev.index, C.byref(out), _stream(stream)))
    return out.value


_PLANS = {}
_PLANS_LOCK = threading.Lock()
_MAX_PLANS = 16


_LAST = [None, None]  # (key of the last lookup with this radii object, plan)


def get_plan(radii, n, batch=1, m0=0, m1=None, device=None, engine=0, fast=0):
    """Cached plan for (device, N, radii, shard, engine, fast) with max_batch >= batch."""
    # fast path: the same radii tuple object as the previous call (a grid's
    # radii) skips hashing M floats
    last_key, last_plan = _LAST
    fast = int(fast)
    if (last_key is not None and last_key[0] is radii and last_key[1:] ==
            (n, m0, m1, device, engine, fast) and last_plan.max_batch >= batch and
            last_plan.handle is not None and
            (device is not None or last_plan.device.index == torch.cuda.current_device())):
        return last_plan
    p = _get_plan(radii, n, batch, m0, m1, device, engine, fast)
    _LAST[0], _LAST[1] = (radii, n, m0, m1, device, engine, fast), p
    return p


def _get_plan(radii, n, batch, m0, m1, device, engine, fast):
    dev = require_cuda(device)
    if not (type(radii) is tuple and all(type(r) is float for r in radii[:1])):
        radii = tuple(float(r) for r in radii)
    key = (dev.index, int(n), radii, int(m0), m1, int(engine), fast)
    with _PLANS_LOCK:
        p = _PLANS.get(key)
        if p is None or p.max_batch < batch:
            if p is not None:
                del _PLANS[key]
            if len(_PLANS) >= _MAX_PLANS:
                _PLANS.pop(next(iter(_PLANS)))
            p = Plan(radii, n, m0=m0, m1=m1, max_batch=max(int(batch), 1), device=dev.index,
                     engine=engine, fast=fast)
            _PLANS[key] = p
        return p
