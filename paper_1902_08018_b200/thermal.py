"""Per-millisecond thermal update on the B200 (thermal.py:81-140 of the
reference): T_{k+1} = fp32(A64 T_k + B u_k), S_{k+1} = fp32(P64 T_{k+1}).

CSR values are widened to binary64 once (thermal.py:101-102) and each row is
accumulated in CSR order like scipy's csr_matvec, so results are bit-identical
to the reference (tests/test_thermal_gpu.py).  numpy in -> numpy out, CUDA
tensors in -> CUDA tensors out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionError, NonFiniteError, WhffError


class DeviceCSR:
    """CSR operator resident on the device with binary64 values."""

    def __init__(self, matrix, device="cuda"):
        torch = _lib.require_cuda()
        if isinstance(matrix, DeviceCSR):
            self.__dict__.update(matrix.__dict__)
            return
        m = matrix.tocsr()
        self.shape = m.shape
        self.nnz = int(m.nnz)
        self.indptr = torch.from_numpy(np.ascontiguousarray(m.indptr, np.int64)).to(device)
        self.indices = torch.from_numpy(np.ascontiguousarray(m.indices, np.int32)).to(device)
        self.data = torch.from_numpy(np.ascontiguousarray(m.data, np.float64)).to(device)

    @property
    def bytes(self):
        return self.indptr.numel() * 8 + self.indices.numel() * 4 + self.data.numel() * 8


def _dev_vec(x):
    torch = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float32).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda(), False


def _check_vector(name, v, n):
    """thermal.py:91-95."""
    from .codec import find_nonfinite
    if tuple(v.shape) != (n,):
        raise DimensionError(f"{name} has shape {tuple(v.shape)}, expected ({n},)")
    bad = find_nonfinite(v)
    if bad is not None:
        raise NonFiniteError(name, bad)


def csr_matvec(A, x, b=None, u=None, out=None):
    """y = fp32(A64 x [+ b*u]) on device tensors, no checks (hot path)."""
    torch = _lib.require_cuda()
    if out is None:
        out = torch.empty(A.shape[0], dtype=torch.float32, device=x.device)
    _lib.call("whff_csr_matvec", _lib.ptr(A.indptr), _lib.ptr(A.indices), _lib.ptr(A.data),
              A.shape[0], _lib.ptr(x), _lib.ptr(b), _lib.ptr(u), _lib.ptr(out), _lib.cur_stream())
    return out


def thermal_step(A64, B, T_k, u_k):
    """thermal.py:98-109."""
    A = A64 if isinstance(A64, DeviceCSR) else DeviceCSR(A64)
    n = A.shape[0]
    t, dev = _dev_vec(T_k)
    u, _ = _dev_vec(u_k)
    b, _ = _dev_vec(B)
    _check_vector("T_k", t, n)
    _check_vector("u_k", u, n)
    if tuple(b.shape) != (n,):
        # the reference's B.astype(f64) * u fails to broadcast (thermal.py:107)
        raise DimensionError(f"B has shape {tuple(b.shape)}, expected ({n},)")
    y = csr_matvec(A, t, b, u)
    return y if dev else y.cpu().numpy()


def thermal_interpolate(P64, T_next):
    """thermal.py:112-117."""
    P = P64 if isinstance(P64, DeviceCSR) else DeviceCSR(P64)
    t, dev = _dev_vec(T_next)
    if P.shape[1] != t.shape[0]:
        raise DimensionError(
            f"interpolation shapes differ: P is {P.shape}, T is {tuple(t.shape)}")
    y = csr_matvec(P, t)
    return y if dev else y.cpu().numpy()


def source_term_device(footprint, dark, dose, out=None):
    """thermal.py:81-88: u = fp32(dose) * footprint + dark (dark step: footprint None)."""
    torch = _lib.require_cuda()
    if out is None:
        out = torch.empty_like(dark)
    _lib.call("whff_source_term", _lib.ptr(footprint), _lib.ptr(dark), float(np.float32(dose)),
              dark.numel(), _lib.ptr(out), _lib.cur_stream())
    return out


@dataclass
class ThermalState:
    """thermal.py:18-28, device resident."""
    k: int
    temperatures: object      # (T,) float32 CUDA tensor
    interpolated: object      # (S,) float32 CUDA tensor

    @classmethod
    def initial(cls, model, S=None):
        """thermal.py:25-28: ``initial(model)`` (anything with ``.T`` and
        ``.S``, the reference's WaferModel included); ``initial(T, S)`` also
        accepted."""
        torch = _lib.require_cuda()
        T = model if S is not None else model.T
        S = S if S is not None else model.S
        return cls(0, torch.zeros(int(T), dtype=torch.float32, device="cuda"),
                   torch.zeros(int(S), dtype=torch.float32, device="cuda"))


class HeatLoad:
    """thermal.py:31-59: dark-phase load plus per-(field, slit) illumination
    footprints (host arrays; DeviceHeatLoad holds the device copy)."""

    def __init__(self, dark_load, light_footprints, dose_scale=1.0):
        dark_load = np.asarray(dark_load, dtype=np.float32)
        bad = np.flatnonzero(~np.isfinite(dark_load))
        if bad.size:
            raise NonFiniteError("dark_load", int(bad[0]))
        self.dark_load = dark_load
        self._footprints = {}
        for key, fp in light_footprints.items():
            fp = np.asarray(fp, dtype=np.float32)
            bad = np.flatnonzero(~np.isfinite(fp))
            if bad.size:
                raise NonFiniteError(f"light_load{key}", int(bad[0]))
            if (fp < 0).any():
                raise WhffError(f"light footprint {key} has negative entries")
            self._footprints[key] = fp
        self.dose_scale = float(dose_scale)

    def light_load(self, field_id, slit_id):
        try:
            return self._footprints[(field_id, slit_id)]
        except KeyError:
            raise WhffError(f"no light footprint for field {field_id} slit {slit_id}") from None

    @property
    def footprints(self):
        return dict(self._footprints)


def synthetic_heatload(model, seed=0, dose_scale=1.0, cooling=1e-3):
    """thermal.py:62-78 (formulas and rng order in synth.heatload)."""
    n_slits = {model.n_slits(f) for f in range(model.n_fields)}
    if len(n_slits) != 1:
        raise WhffError("synthetic_heatload expects the same slit count in every field")
    dark, fps, dose = synth_heatload(model.spec, model.n_fields, n_slits.pop(), seed=seed,
                                     dose_scale=dose_scale, cooling=cooling)
    return HeatLoad(dark, fps, dose)


def synth_heatload(*a, **k):
    from .synth import heatload
    return heatload(*a, **k)


class DeviceHeatLoad:
    """Device copy of a reference HeatLoad (thermal.py:31-59)."""

    def __init__(self, dark_load, light_footprints, dose_scale=1.0):
        torch = _lib.require_cuda()
        self.dark = torch.from_numpy(np.ascontiguousarray(dark_load, np.float32)).cuda()
        self.footprints = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda()
                           for k, v in light_footprints.items()}
        self.dose_scale = float(dose_scale)

    def source(self, field_id, phase, slit_id=None, out=None):
        if phase == "dark":
            return source_term_device(None, self.dark, 0.0, out)
        if phase != "light":
            raise WhffError(f"step phase must be light or dark, got {phase!r}")
        try:
            fp = self.footprints[(field_id, slit_id)]
        except KeyError:
            raise WhffError(f"no light footprint for field {field_id} slit {slit_id}") from None
        return source_term_device(fp, self.dark, self.dose_scale, out)


def source_term(load, field_id, phase, slit_id=None):
    """thermal.py:81-88 on the device: u_k for one schedule step (binary32
    fp32(dose) * footprint + dark, or the dark load); returns numpy."""
    if phase not in ("light", "dark"):
        raise WhffError(f"step phase must be light or dark, got {phase!r}")
    fps = {} if phase == "dark" else {(field_id, slit_id): load.light_load(field_id, slit_id)}
    dev = DeviceHeatLoad(load.dark_load, fps, load.dose_scale)
    return dev.source(field_id, phase, slit_id).cpu().numpy()


def run_field_thermal(model, field_schedule, load, state, A=None, P=None, B=None):
    """thermal.py:120-140 on the device: advance `state` (a device
    ThermalState) across one field, yielding (k, phase, slit, S_next) with
    S_next a CUDA tensor for light steps and None for dark ones.  A, P, B
    (DeviceCSR / tensor) may be passed to reuse uploaded operators."""
    torch = _lib.require_cuda()
    A = A if A is not None else DeviceCSR(model.A_f64())
    P = P if P is not None else DeviceCSR(model.P_f64())
    B = B if B is not None else torch.from_numpy(np.ascontiguousarray(model.B, np.float32)).cuda()
    n_slits = model.n_slits(field_schedule.field_id)
    keys = {(field_schedule.field_id, field_schedule.slit_for_light_step(i, n_slits))
            for i in range(field_schedule.t_l)}
    dev = DeviceHeatLoad(load.dark_load, {k: load.light_load(*k) for k in keys}, load.dose_scale)
    # a reference (numpy) ThermalState: advance a device copy, write back per step
    host_state = isinstance(state.temperatures, np.ndarray)
    T_cur = (torch.from_numpy(np.ascontiguousarray(state.temperatures, np.float32)).cuda()
             if host_state else state.temperatures)
    u = torch.empty_like(T_cur)
    for i in range(field_schedule.t_l + field_schedule.t_d):
        if i < field_schedule.t_l:
            phase, slit = "light", field_schedule.slit_for_light_step(i, n_slits)
        else:
            phase, slit = "dark", None
        dev.source(field_schedule.field_id, phase, slit, out=u)
        t_next = csr_matvec(A, T_cur, B, u)
        s_next = csr_matvec(P, t_next)
        T_cur = t_next
        state.k += 1
        if host_state:
            state.temperatures = t_next.cpu().numpy()
            state.interpolated = s_next.cpu().numpy()
        else:
            state.temperatures = t_next
            state.interpolated = s_next
        yield state.k, phase, slit, (s_next if phase == "light" else None)
