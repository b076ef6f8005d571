"""B200-native forward model of arXiv 2306.00271 (manybeam) — Python host mirror.

This module mirrors the reference C++ library's forward-model interface
(/root/reference/proj/core/include/manybeam/*.hpp) over the C-ABI of
``libmanybeam_b200.so`` (include/manybeam_b200.h):

    RodSet.build / RodSet.build_first        rods.hpp:23-47
    PotentialField.zero / gaussian_layers /
        tabulated / atoms                     potential.hpp:35-61 (+ atoms extension)
    StepperSpec.rk4 / sp4 / sp6 / splitting   proposed.hpp:23-43
    AngleGrid.validated, SweepOptions         sweep.hpp:17-32
    rocking_curve(field, rods, gamma, grid, opts) -> RockingCurve   sweep.hpp:37-38
    solve_batch(...)                           batched structures (no reference analogue)
    curve_error                               curve.hpp:38

Errors are raised with the reference's exception taxonomy (types.hpp:20-62).
There is no CPU fallback: the shared library must be present and a B200
(sm_100) device visible, otherwise every solve raises CudaError.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("MB_LIB") or os.path.join(_HERE, "libmanybeam_b200.so")

# ----------------------------------------------------------------- errors


class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class SolverError(Error):
    pass


class SingularMatrixError(SolverError):
    pass


class BreakdownError(SolverError):
    def __init__(self, msg, step=None):
        super().__init__(msg)
        self.step = step


class ConvergenceError(SolverError):
    pass


class DomainError(SolverError):
    pass


class IoError(Error):
    """types.hpp IoError: curve CSV read/write failures."""


class CompareError(Error):
    pass


class CudaError(Error):
    pass


MB_OK, MB_ERR_CONFIG, MB_ERR_SOLVER, MB_ERR_SINGULAR, MB_ERR_BREAKDOWN = 0, 1, 2, 3, 4
MB_ERR_CONVERGENCE, MB_ERR_DOMAIN, MB_ERR_CUDA, MB_ERR_ARG = 5, 6, 7, 8
_ERRORS = {
    MB_ERR_CONFIG: ConfigError,
    MB_ERR_SOLVER: SolverError,
    MB_ERR_SINGULAR: SingularMatrixError,
    MB_ERR_BREAKDOWN: BreakdownError,
    MB_ERR_CONVERGENCE: ConvergenceError,
    MB_ERR_DOMAIN: DomainError,
    MB_ERR_CUDA: CudaError,
    MB_ERR_ARG: ValueError,
}

# ----------------------------------------------------------------- C structs


class _Lattice(C.Structure):
    _fields_ = [("a1", C.c_double * 2), ("a2", C.c_double * 2)]


class _Rods(C.Structure):
    _fields_ = [("n", C.c_int), ("k", C.c_void_p), ("m", C.c_void_p), ("ndiff", C.c_int),
                ("diff", C.c_void_p), ("diff_m", C.c_void_p), ("diff_index", C.c_void_p)]


class _Field(C.Structure):
    _fields_ = [("kind", C.c_int), ("z_bottom", C.c_double), ("has_bulk_period", C.c_int),
                ("bulk_period", C.c_double), ("nlayers", C.c_int), ("layers", C.c_void_p),
                ("ngrid", C.c_int), ("z_grid", C.c_void_p), ("nentries", C.c_int), ("entry_dm", C.c_void_p),
                ("entry_values", C.c_void_p), ("natoms", C.c_int), ("atom_xyz", C.c_void_p),
                ("atom_species", C.c_void_p), ("atom_B", C.c_void_p), ("nspecies", C.c_int),
                ("ff_a", C.c_void_p), ("ff_b", C.c_void_p), ("cell_area", C.c_double),
                ("gamma_L", C.c_double), ("particle_sign", C.c_double), ("absorption", C.c_double)]


class _Stepper(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("variant", C.c_int), ("ndrift", C.c_int), ("drift", C.c_void_p),
                ("nkick", C.c_int), ("kick", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("dz", C.c_double), ("slices", C.c_long), ("rhst_threshold", C.c_double),
                ("residual_check", C.c_int), ("fsal", C.c_int), ("path", C.c_int)]


class _Pair(C.Structure):
    _fields_ = [("structure", C.c_int), ("theta0_deg", C.c_double), ("theta1_deg", C.c_double)]


POINT_STATUS_DTYPE = np.dtype([("code", np.int32), ("step", np.int32), ("rhst", np.int32),
                               ("rhst_pivoting", np.int32)])
POINT_OK, POINT_NONFINITE, POINT_RHST, POINT_EXTRACTION = 0, 1, 2, 3

_lib = None


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load the C-ABI library (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise CudaError(f"{_LIB_PATH} is missing: build it with `make -C {_HERE}` "
                            "(no CPU fallback exists)")
        L = C.CDLL(_LIB_PATH)
        L.mb_last_error.restype = C.c_char_p
        L.mb_rods_build.argtypes = [C.POINTER(_Lattice), C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.mb_beam_from_energy.argtypes = [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.mb_stepper_by_name.argtypes = [C.c_char_p, C.POINTER(_Stepper)]
        L.mb_context_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.mb_context_destroy.argtypes = [C.c_void_p]
        L.mb_context_create_multi.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.mb_context_device_count.argtypes = [C.c_void_p]
        L.mb_device_ok.argtypes = [C.c_int]
        L.mb_plan_create.argtypes = [C.c_void_p, C.POINTER(_Rods), C.POINTER(_Field), C.c_int, C.c_double,
                                     C.POINTER(_Pair), C.c_long, C.POINTER(_Stepper), C.POINTER(_Options),
                                     C.POINTER(C.c_void_p)]
        L.mb_plan_create_seeded.argtypes = [C.c_void_p, C.POINTER(_Rods), C.POINTER(_Field), C.c_int, C.c_double,
                                            C.POINTER(_Pair), C.c_long, C.POINTER(_Stepper), C.POINTER(_Options),
                                            C.c_void_p, C.c_long, C.POINTER(C.c_void_p)]
        L.mb_plan_execute.argtypes = [C.c_void_p, C.c_void_p]
        L.mb_plan_results.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.mb_plan_timing.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.mb_plan_info.argtypes = [C.c_void_p, C.POINTER(C.c_long), C.POINTER(C.c_int), C.POINTER(C.c_long),
                                   C.POINTER(C.c_int), C.POINTER(C.c_long)]
        L.mb_plan_destroy.argtypes = [C.c_void_p]
        L.mb_plan_profile.argtypes = [C.c_void_p, C.c_void_p]
        L.mb_plan_node_heights.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
        L.mb_plan_gamma.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.mb_plan_coefficients.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_long]
        L.mb_rocking_curve.argtypes = [C.c_void_p, C.POINTER(_Field), C.POINTER(_Rods), C.c_double, C.c_void_p,
                                       C.c_int, C.c_void_p, C.c_int, C.POINTER(_Stepper), C.POINTER(_Options),
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _check(rc, status=None):
    if rc == MB_OK:
        return
    msg = lib().mb_last_error().decode()
    exc = _ERRORS.get(rc, Error)
    if exc is BreakdownError:
        step = None
        if status is not None:
            bad = np.nonzero(status["code"] != POINT_OK)[0]
            if len(bad):
                step = int(status["step"][bad[0]])
        raise BreakdownError(msg, step)
    raise exc(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- geometry
@dataclass
class Lattice2D:
    """2-D surface lattice (rods.hpp:10-17)."""
    a1: tuple
    a2: tuple

    def b1(self):
        det = self.a1[0] * self.a2[1] - self.a1[1] * self.a2[0]
        return (2 * math.pi * self.a2[1] / det, -2 * math.pi * self.a2[0] / det)

    def b2(self):
        det = self.a1[0] * self.a2[1] - self.a1[1] * self.a2[0]
        return (-2 * math.pi * self.a1[1] / det, 2 * math.pi * self.a1[0] / det)

    @property
    def area(self):
        return abs(self.a1[0] * self.a2[1] - self.a1[1] * self.a2[0])

    @staticmethod
    def hexagonal(a):
        return Lattice2D((a, 0.0), (a * math.cos(2 * math.pi / 3), a * math.sin(2 * math.pi / 3)))

    @staticmethod
    def rectangular(a, b):
        return Lattice2D((a, 0.0), (0.0, b))


class RodSet:
    """Reciprocal rods sorted by (||k||, kx, ky) with the deduplicated
    difference table (rods.hpp:23-47)."""

    def __init__(self, lattice, k, m, diff, diff_m, diff_index, cutoff):
        self.lattice, self.k, self.m = lattice, k, m
        self.diff, self.diff_m, self.diff_index, self.cutoff = diff, diff_m, diff_index, cutoff

    @staticmethod
    def _build(lattice, cutoff, first_n):
        L = lib()
        lat = _Lattice((C.c_double * 2)(*lattice.a1), (C.c_double * 2)(*lattice.a2))
        n, nd = C.c_int(), C.c_int()
        _check(L.mb_rods_build(C.byref(lat), float(cutoff), int(first_n), C.byref(n), C.byref(nd),
                               None, None, None, None, None, 0, 0))
        k = np.zeros((n.value, 2))
        m = np.zeros((n.value, 2), np.int32)
        diff = np.zeros((nd.value, 2))
        diff_m = np.zeros((nd.value, 2), np.int32)
        di = np.zeros((n.value, n.value), np.int32)
        _check(L.mb_rods_build(C.byref(lat), float(cutoff), int(first_n), C.byref(n), C.byref(nd), _ptr(k), _ptr(m),
                               _ptr(diff), _ptr(diff_m), _ptr(di), n.value, nd.value))
        c = cutoff if first_n <= 0 else float(np.linalg.norm(k[-1]))
        return RodSet(lattice, k, m, diff, diff_m, di, c)

    @staticmethod
    def build(lattice, cutoff):
        return RodSet._build(lattice, cutoff, 0)

    @staticmethod
    def build_first(lattice, n):
        """EXTENSION: the first n rods of the reference order."""
        if n < 1:
            raise ConfigError("rod count must be >= 1")
        return RodSet._build(lattice, 0.0, n)

    def size(self):
        return len(self.k)

    def diff_count(self):
        return len(self.diff)

    def _c(self):
        return _Rods(self.size(), _ptr(self.k), _ptr(self.m), self.diff_count(), _ptr(self.diff), _ptr(self.diff_m),
                     _ptr(self.diff_index))

    def labels(self):
        return [f"({a};{b})" for a, b in self.m]


def beam_from_energy(energy_ev):
    """EXTENSION: relativistic (gamma [1/A], gamma_L) from kinetic energy (eV)."""
    g, gl = C.c_double(), C.c_double()
    _check(lib().mb_beam_from_energy(float(energy_ev), C.byref(g), C.byref(gl)))
    return g.value, gl.value


# ----------------------------------------------------------------- potential
MB_FIELD_ZERO, MB_FIELD_GAUSSIAN_LAYERS, MB_FIELD_TABULATED, MB_FIELD_ATOMS = 0, 1, 2, 3


@dataclass
class GaussianLayer:
    z_center: float = 0.0
    amplitude: float = 0.0
    sigma_xy: float = 1.0
    sigma_z: float = 1.0
    absorption: float = 0.0


class PotentialField:
    """Laterally periodic scattering potential (potential.hpp:35-61) plus the
    atom-list model."""

    def __init__(self, kind, z_bottom, **kw):
        self.kind, self.z_bottom = kind, float(z_bottom)
        self.bulk_period = kw.pop("bulk_period", None)
        self.__dict__.update(kw)

    @staticmethod
    def zero(z_bottom):
        return PotentialField(MB_FIELD_ZERO, z_bottom)

    @staticmethod
    def gaussian_layers(z_bottom, layers, bulk_period=None):
        arr = np.array([[l.z_center, l.amplitude, l.sigma_xy, l.sigma_z, l.absorption] if isinstance(l, GaussianLayer)
                        else list(l) for l in layers], dtype=np.float64).reshape(-1, 5)
        return PotentialField(MB_FIELD_GAUSSIAN_LAYERS, z_bottom, layers=arr, bulk_period=bulk_period)

    @staticmethod
    def tabulated(z_bottom, z_grid, entries, bulk_period=None):
        """entries: list of ((dm1, dm2), complex values per grid point)."""
        z = np.ascontiguousarray(z_grid, dtype=np.float64)
        dm = np.array([e[0] for e in entries], dtype=np.int32).reshape(-1, 2)
        vals = np.array([np.asarray(e[1], dtype=np.complex128) for e in entries]).reshape(len(entries), -1)
        if vals.shape[1] != len(z) and len(entries):
            raise ConfigError("potential: tabulated entry sample count does not match the z grid")
        v = np.ascontiguousarray(vals).view(np.float64).reshape(len(entries), len(z), 2)
        return PotentialField(MB_FIELD_TABULATED, z_bottom, z_grid=z, entry_dm=dm, entry_values=v,
                              bulk_period=bulk_period)

    @staticmethod
    def atoms(z_bottom, xyz, species, B, ff_a, ff_b, cell_area, gamma_L, particle_sign, absorption=0.1,
              bulk_period=None):
        """EXTENSION: atom list (Cartesian A), species index, Debye-Waller B (A^2),
        4-Gaussian form factors ff_a (A) / ff_b (A^2) per species."""
        return PotentialField(MB_FIELD_ATOMS, z_bottom,
                              xyz=np.ascontiguousarray(xyz, np.float64).reshape(-1, 3),
                              species=np.ascontiguousarray(species, np.int32).reshape(-1),
                              B=np.ascontiguousarray(B, np.float64).reshape(-1),
                              ff_a=np.ascontiguousarray(ff_a, np.float64).reshape(-1, 4),
                              ff_b=np.ascontiguousarray(ff_b, np.float64).reshape(-1, 4),
                              cell_area=float(cell_area), gamma_L=float(gamma_L),
                              particle_sign=float(particle_sign), absorption=float(absorption),
                              bulk_period=bulk_period)

    def _c(self):
        f = _Field()
        f.kind, f.z_bottom = self.kind, self.z_bottom
        f.has_bulk_period = int(self.bulk_period is not None)
        f.bulk_period = float(self.bulk_period or 0.0)
        if self.kind == MB_FIELD_GAUSSIAN_LAYERS:
            f.nlayers, f.layers = len(self.layers), _ptr(self.layers)
        elif self.kind == MB_FIELD_TABULATED:
            f.ngrid, f.z_grid = len(self.z_grid), _ptr(self.z_grid)
            f.nentries, f.entry_dm, f.entry_values = len(self.entry_dm), _ptr(self.entry_dm), _ptr(self.entry_values)
        elif self.kind == MB_FIELD_ATOMS:
            f.natoms, f.atom_xyz, f.atom_species, f.atom_B = len(self.xyz), _ptr(self.xyz), _ptr(self.species), _ptr(self.B)
            f.nspecies, f.ff_a, f.ff_b = len(self.ff_a), _ptr(self.ff_a), _ptr(self.ff_b)
            f.cell_area, f.gamma_L = self.cell_area, self.gamma_L
            f.particle_sign, f.absorption = self.particle_sign, self.absorption
        return f


# ----------------------------------------------------------------- stepper
class StepperSpec:
    """One-step integrator (proposed.hpp:23-43)."""
    RK4, SPLITTING, CONVENTIONAL = 0, 1, 2
    ABA, BAB = 0, 1

    def __init__(self, name, algorithm, variant=1, drift=(), kick=()):
        self.name, self.algorithm, self.variant = name, algorithm, variant
        self.drift = np.ascontiguousarray(drift, np.float64)
        self.kick = np.ascontiguousarray(kick, np.float64)

    @staticmethod
    def by_name(name):
        s = _Stepper()
        _check(lib().mb_stepper_by_name(name.encode(), C.byref(s)))
        if s.algorithm in (StepperSpec.RK4, StepperSpec.CONVENTIONAL):
            return StepperSpec(name, s.algorithm)
        drift = np.ctypeslib.as_array(C.cast(s.drift, C.POINTER(C.c_double)), (s.ndrift,)).copy()
        kick = np.ctypeslib.as_array(C.cast(s.kick, C.POINTER(C.c_double)), (s.nkick,)).copy()
        return StepperSpec(name, StepperSpec.SPLITTING, s.variant, drift, kick)

    @staticmethod
    def rk4():
        return StepperSpec.by_name("rk4")

    @staticmethod
    def sp4():
        return StepperSpec.by_name("sp4")

    @staticmethod
    def sp6():
        return StepperSpec.by_name("sp6")

    @staticmethod
    def splitting(name, variant, drift, kick):
        return StepperSpec(name, StepperSpec.SPLITTING, variant, drift, kick)

    def kicks_per_step(self):
        return 4 if self.algorithm == StepperSpec.RK4 else len(self.kick)

    def _c(self):
        return _Stepper(self.algorithm, self.variant, len(self.drift), _ptr(self.drift), len(self.kick), _ptr(self.kick))


# ----------------------------------------------------------------- sweep
@dataclass
class AngleGrid:
    theta0: list
    theta1: list

    @staticmethod
    def validated(theta0, theta1):  # sweep.cpp:18-33
        theta0, theta1 = [float(t) for t in theta0], [float(t) for t in theta1]
        if not theta0:
            raise ConfigError("angle grid: theta0 list is empty")
        if not theta1:
            raise ConfigError("angle grid: theta1 list is empty")
        if any(not (0.0 < t < 90.0) for t in theta0):
            raise ConfigError("angle grid: glancing angles must lie in (0, 90) degrees")
        if any(not (b > a) for a, b in zip(theta0, theta0[1:])):
            raise ConfigError("angle grid: theta0 must be strictly increasing")
        if any(not math.isfinite(t) for t in theta1):
            raise ConfigError("angle grid: theta1 must be finite")
        return AngleGrid(theta0, theta1)

    def rows(self):
        return len(self.theta0) * len(self.theta1)


@dataclass
class SweepOptions:
    """sweep.hpp:26-32 for the stepper methods (+ device options)."""
    method: str = "sp6"
    dz: float = 0.01
    slices: int = 0            # EXTENSION: >0 fixes the slice count
    rhst_threshold: float = 1000.0
    residual_check: bool = True
    fsal: bool = False
    stepper: Optional[StepperSpec] = None  # custom splitting coefficients
    path: int = 0              # 0 auto, 1 resident on-chip kernel, 2 batched large-N kernels,
    #                            3 cluster kernel, 4 cluster kernel as cooperative groups

    def _stepper(self):
        return self.stepper if self.stepper is not None else StepperSpec.by_name(self.method)

    def _c(self):
        return _Options(float(self.dz), int(self.slices), float(self.rhst_threshold), int(bool(self.residual_check)),
                        int(bool(self.fsal)), int(self.path))


@dataclass
class RockingCurve:
    """curve.hpp:19-31 (+ rho, status)."""
    theta0: list
    theta1: list
    eta: np.ndarray
    rod_labels: list
    method: str
    dz: float
    rhst_threshold: float
    solve_seconds: float = 0.0
    rho: Optional[np.ndarray] = None
    status: Optional[np.ndarray] = None

    def rows(self):
        return len(self.theta0)

    def rod_count(self):
        return self.eta.shape[1]


class Context:
    """A device context (streams + pooled device memory). With `devices`
    (a list, repeats allowed) one context drives several GPUs: plans split
    their pairs over them (mb_context_create_multi)."""

    def __init__(self, device=0, devices=None):
        self._h = C.c_void_p()
        if devices is not None:
            arr = (C.c_int * len(devices))(*[int(d) for d in devices])
            _check(lib().mb_context_create_multi(arr, len(devices), C.byref(self._h)))
            self.device, self.devices = int(devices[0]), list(devices)
        else:
            _check(lib().mb_context_create(int(device), C.byref(self._h)))
            self.device, self.devices = device, [device]

    def close(self):
        if self._h:
            lib().mb_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Plan:
    """Batched solve over (structure, angle) pairs sharing rods, gamma and
    slicing: create (host prep + uploads) / execute (K1 + K2 on the device) /
    results (D2H). r_init: optional caller-supplied R_init of solve_proposed
    (proposed.hpp:98-102), one (n, n) complex matrix shared by every pair or
    (npairs, n, n); it replaces the bulk seed."""

    def __init__(self, rods, fields, gamma, pairs, opts, ctx=None, r_init=None):
        self.ctx = ctx or default_context()
        self.rods, self.fields = rods, list(fields)
        self.pairs = np.asarray(pairs)
        self.n = rods.size()
        st = opts._stepper()
        self._keep = [rods._c(), [f._c() for f in self.fields], st._c(), opts._c(), st]
        crods, cfields, cst, copt, _ = self._keep
        farr = (_Field * len(cfields))(*cfields)
        parr = (_Pair * len(self.pairs))(*[_Pair(int(s), float(t0), float(t1)) for s, t0, t1 in self.pairs])
        self._arrays = (farr, parr)
        self._h = C.c_void_p()
        if r_init is None:
            _check(lib().mb_plan_create(self.ctx._h, C.byref(crods), farr, len(cfields), float(gamma), parr,
                                        len(self.pairs), C.byref(cst), C.byref(copt), C.byref(self._h)))
        else:
            R = np.ascontiguousarray(r_init, np.complex128)
            if R.ndim == 2:
                R = R[None]
            if R.ndim != 3 or R.shape[1:] != (self.n, self.n):
                raise SolverError("R_init has wrong dimensions")  # proposed.cpp:126
            _check(lib().mb_plan_create_seeded(self.ctx._h, C.byref(crods), farr, len(cfields), float(gamma), parr,
                                               len(self.pairs), C.byref(cst), C.byref(copt), _ptr(R), R.shape[0],
                                               C.byref(self._h)))
        self.npairs = len(self.pairs)

    def execute(self, stream=None):
        _check(lib().mb_plan_execute(self._h, C.c_void_p(stream) if stream else None))

    def results(self, want_rho=True, raise_on_error=True):
        eta = np.zeros((self.npairs, self.n))
        rho = np.zeros((self.npairs, self.n), np.complex128) if want_rho else None
        status = np.zeros(self.npairs, POINT_STATUS_DTYPE)
        rc = lib().mb_plan_results(self._h, _ptr(eta), _ptr(rho), _ptr(status))
        if raise_on_error:
            _check(rc, status)
        return eta, rho, status

    def timing(self):
        t, p, q, n = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        _check(lib().mb_plan_timing(self._h, C.byref(t), C.byref(p), C.byref(q), C.byref(n)))
        return {"ms_total": t.value, "ms_potential": p.value, "ms_propagate": q.value, "launches": n.value}

    def info(self):
        s, d, b, npad, h2d = C.c_long(), C.c_int(), C.c_long(), C.c_int(), C.c_long()
        _check(lib().mb_plan_info(self._h, C.byref(s), C.byref(d), C.byref(b), C.byref(npad), C.byref(h2d)))
        return {"slots": s.value, "ndiff": d.value, "coef_bytes": b.value, "npad": npad.value, "h2d_bytes": h2d.value}

    PHASES = ("table_wait", "gemm", "kick_epilogue", "rhst_gj", "gershgorin", "rhst_other", "surface", "prologue",
              "gj_rows_pre", "gj_pivot", "gj_rows_post", "gj_sync", "slot12", "slot13", "slot14", "slot15")

    def profile(self):
        """per-CTA cycles by phase (MB_PROFILE builds only)."""
        v = np.zeros(16)
        _check(lib().mb_plan_profile(self._h, _ptr(v)))
        return dict(zip(self.PHASES, v.tolist()))

    # parity hooks (EXTENSION): what plan creation / K1 produced
    def node_heights(self):
        z = np.zeros(self.info()["slots"])
        _check(lib().mb_plan_node_heights(self._h, _ptr(z), len(z)))
        return z

    def gamma(self, pair):
        gd = np.zeros(self.n, np.complex128)
        gi = np.zeros(self.n, np.complex128)
        g2 = np.zeros(self.n)
        s0 = C.c_double()
        _check(lib().mb_plan_gamma(self._h, int(pair), _ptr(gd), _ptr(gi), _ptr(g2), C.byref(s0)))
        return gd, gi, g2, s0.value

    def coefficients(self, structure=0):
        inf = self.info()
        c = np.zeros((inf["slots"], inf["ndiff"]), np.complex128)
        _check(lib().mb_plan_coefficients(self._h, int(structure), _ptr(c), 2 * c.size))
        return c

    def close(self):
        if self._h:
            lib().mb_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_batch(fields, rods, gamma, pairs, opts, ctx=None, want_rho=True, r_init=None):
    """Batched structures: pairs = [(structure_index, theta0_deg, theta1_deg)].
    Returns (eta[npairs][n], rho, status)."""
    plan = Plan(rods, fields, gamma, pairs, opts, ctx, r_init=r_init)
    try:
        plan.execute()
        return plan.results(want_rho)
    finally:
        plan.close()


def solve_proposed(field, rods, gamma, theta0_deg, theta1_deg, opts, r_init=None, ctx=None):
    """solve_proposed (proposed.hpp:98-102, proposed.cpp:293-309) for one beam
    direction: rho0, the first column of R at the surface, from the state
    seeded with R_init (zero when None) at z_bottom. Returns (rho0, rhst_count);
    breakdowns raise like the reference (BreakdownError with the step)."""
    _, rho, st = solve_batch([field], rods, gamma, [(0, theta0_deg, theta1_deg)], opts, ctx, True, r_init)
    return rho[0], int(st["rhst"][0])


def rocking_curve(field, rods, gamma, grid, opts, ctx=None):
    """sweep.hpp:37-38 — rows theta1-major, theta0 inner (sweep.cpp:90-91)."""
    import time
    ctx = ctx or default_context()
    t0 = time.perf_counter()
    th0 = np.ascontiguousarray(grid.theta0, np.float64)
    th1 = np.ascontiguousarray(grid.theta1, np.float64)
    rows = len(th0) * len(th1)
    n = rods.size()
    eta = np.zeros((rows, n))
    rho = np.zeros((rows, n), np.complex128)
    status = np.zeros(rows, POINT_STATUS_DTYPE)
    st = opts._stepper()
    cf, cr, cs, co = field._c(), rods._c(), st._c(), opts._c()
    rc = lib().mb_rocking_curve(ctx._h, C.byref(cf), C.byref(cr), float(gamma), _ptr(th0), len(th0), _ptr(th1),
                                len(th1), C.byref(cs), C.byref(co), _ptr(eta), _ptr(rho), _ptr(status))
    _check(rc, status)
    return RockingCurve([t0_ for _ in th1 for t0_ in th0], [t1_ for t1_ in th1 for _ in th0], eta, rods.labels(),
                        opts.method if opts.stepper is None else opts.stepper.name, opts.dz, opts.rhst_threshold,
                        time.perf_counter() - t0, rho, status)


def curve_error(candidate, reference):
    """curve.cpp:22-41: max_rows ||d eta|| / max_rows ||eta_ref||."""
    a, b = np.asarray(candidate.eta), np.asarray(reference.eta)
    if a.shape[0] != b.shape[0]:
        raise CompareError("curve_error: row count mismatch")
    if a.shape[1] != b.shape[1]:
        raise CompareError("curve_error: rod count mismatch")
    if (np.abs(np.subtract(candidate.theta0, reference.theta0)) > 1e-12).any() or \
            (np.abs(np.subtract(candidate.theta1, reference.theta1)) > 1e-12).any():
        raise CompareError("curve_error: angle grids differ")
    num = np.linalg.norm(a - b, axis=1).max()
    den = np.linalg.norm(b, axis=1).max()
    if num == 0.0:
        return 0.0
    if den == 0.0:
        return math.inf
    return float(num / den)


def device_available(device=0):
    try:
        return bool(lib().mb_device_ok(int(device)))
    except Exception:
        return False

# ---------------------------------------------------------------- curve CSV
# The reference's wire format (csvio.cpp:65-149):
# "# key: value" metadata, header theta0,theta1,eta(m1;m2)..., every number
# as %.14E; byte-identical to the C++ writer in include/manybeam_b200.hpp.
def format_full(v):
    return ("%.14E" % float(v)).replace(",", ".")


def write_curve_csv(path, curve):
    lines = ["# manybeam-curve v1", f"# method: {curve.method}", f"# dz: {format_full(curve.dz)}"]
    if curve.method != "conventional":
        thr = curve.rhst_threshold
        lines.append("# rhst_threshold: " + ("inf" if math.isinf(thr) else format_full(thr)))
    eta = np.asarray(curve.eta)
    lines.append(f"# rods: {eta.shape[1]}")
    lines.append(",".join(["theta0", "theta1"] + [f"eta{l}" for l in curve.rod_labels]))
    for r in range(eta.shape[0]):
        lines.append(",".join([format_full(curve.theta0[r]), format_full(curve.theta1[r])] +
                              [format_full(x) for x in eta[r]]))
    try:
        with open(path, "wb") as f:
            f.write(("\n".join(lines) + "\n").encode())
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def read_curve_csv(path):
    try:
        text = open(path, "rb").read().decode()
    except OSError as e:
        raise IoError(f"cannot open '{path}'") from e
    meta, labels, t0, t1, rows, ncols = {}, None, [], [], [], 0

    def num(f, what):
        if f == "inf":
            return math.inf
        try:
            return float(f)
        except ValueError:
            raise IoError(f"curve csv: bad {what} value '{f}'") from None

    for line in text.splitlines():
        t = line.strip()
        if not t:
            continue
        if t.startswith("#"):
            if ":" in t:
                k, v = t[1:].split(":", 1)
                meta[k.strip()] = v.strip()
            continue
        fields = [x.strip() for x in t.split(",")]
        if labels is None:
            if len(fields) < 3 or fields[0] != "theta0" or fields[1] != "theta1":
                raise IoError("curve csv: expected header starting with theta0,theta1")
            if not all(f.startswith("eta") for f in fields[2:]):
                raise IoError("curve csv: intensity columns must be named eta(...)")
            labels, ncols = [f[3:] for f in fields[2:]], len(fields)
            continue
        if len(fields) != ncols:
            raise IoError(f"curve csv: row has {len(fields)} fields, expected {ncols}")
        t0.append(num(fields[0], "theta0"))
        t1.append(num(fields[1], "theta1"))
        rows.append([num(f, "eta") for f in fields[2:]])
    if labels is None:
        raise IoError("curve csv: missing header row")
    if not rows:
        raise IoError("curve csv: no data rows")
    return RockingCurve(t0, t1, np.array(rows), labels, meta.get("method", ""), num(meta.get("dz", "0"), "dz"),
                        num(meta.get("rhst_threshold", "inf"), "threshold"))


def compare_curve_files(candidate, reference):
    """The reference CLI's `compare` (main.cpp): curve_error of two stored curves."""
    return curve_error(read_curve_csv(candidate), read_curve_csv(reference))
