"""Seeded synthetic workloads for the five BASELINE.json configs.

There is no public dataset for this path (the paper's Si(111)-7x7 inputs are
not in the container); these generators stand in for them
with the shapes, sizes and value distributions BASELINE.json names
(SURVEY.md §8d). Every value derives from a fixed numpy seed, so the oracle
and the device path consume identical inputs.

Potential convention: u = (sign - 0.1 i) V with
sign = +1 for electrons and -1 for positrons, so Im U < 0 (absorbing,
potential.hpp:15-16) for both particles.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

SPECIES_Z = (14, 32)
SPECIES_SEED = 20230601


def form_factors(seed=SPECIES_SEED):
    """4-Gaussian electron form factors per species: a_i ~ U[0.1, 2.0] A,
    b_i ~ U[0.5, 40] A^2 (BASELINE.json config 0)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.1, 2.0, (len(SPECIES_Z), 4))
    b = rng.uniform(0.5, 40.0, (len(SPECIES_Z), 4))
    return a, b


def relativistic(energy_ev):
    """gamma = 2 pi / lambda (1/A) and gamma_L = 1 + E/m0c^2 (same formula as
    mb_beam_from_energy; restated so the generator has no device dependency)."""
    mc2, hc = 510998.95, 12398.419843320026
    lam = hc / math.sqrt(energy_ev * (energy_ev + 2.0 * mc2))
    return 2.0 * math.pi / lam, 1.0 + energy_ev / mc2


@dataclass
class Structure:
    xyz: np.ndarray      # [natoms][3] Cartesian A
    species: np.ndarray  # [natoms] index into SPECIES_Z
    B: np.ndarray        # [natoms] Debye-Waller A^2


@dataclass
class Workload:
    name: str
    a1: tuple
    a2: tuple
    n_rods: int
    energy_ev: float
    particle: str        # "electron" | "positron"
    z_bottom: float
    slices: int
    method: str
    theta0: List[float]
    structures: List[Structure]
    pairs: np.ndarray = None  # [npairs][3]: structure, theta0, theta1 (default: all x all)
    theta1: List[float] = field(default_factory=lambda: [0.0])
    absorption: float = 0.1
    bulk_period: float = None  # bulk seed below z_bottom (compute_bulk_reflection_proposed); None: R_init = 0

    @property
    def cell_area(self):
        return abs(self.a1[0] * self.a2[1] - self.a1[1] * self.a2[0])

    @property
    def gamma(self):
        return relativistic(self.energy_ev)[0]

    @property
    def gamma_L(self):
        return relativistic(self.energy_ev)[1]

    @property
    def sign(self):
        return 1.0 if self.particle == "electron" else -1.0

    def all_pairs(self):
        if self.pairs is not None:
            return self.pairs
        return np.array([(s, t0, t1) for s in range(len(self.structures)) for t1 in self.theta1 for t0 in self.theta0],
                        dtype=object)

    def points(self):
        return len(self.all_pairs())

    def flops_per_point(self, kicks_per_step=None):
        """Algorithmic FP64 flops per point: L * s_eff * 8 N^3:
        s_eff = 4 (rk4), 6 (sp4, FSAL), 11 (sp6, FSAL)."""
        s_eff = {"rk4": 4, "sp4": 6, "sp6": 11}[self.method] if kicks_per_step is None else kicks_per_step
        return float(self.slices) * s_eff * 8.0 * self.n_rods ** 3

    def subset(self, structures=None, theta0=None, slices=None, name=None, z_bottom=None):
        """Smaller case with the same generator (for parity tests); a thinner
        slab (z_bottom) with proportionally fewer slices keeps the step h."""
        w = Workload(name or self.name, self.a1, self.a2, self.n_rods, self.energy_ev, self.particle,
                     z_bottom if z_bottom is not None else self.z_bottom,
                     slices or self.slices, self.method, list(theta0 if theta0 is not None else self.theta0),
                     [self.structures[i] for i in (structures if structures is not None else range(len(self.structures)))],
                     None, list(self.theta1), self.absorption, self.bulk_period)
        return w


def _hex(a):
    return (a, 0.0), (a * math.cos(2 * math.pi / 3), a * math.sin(2 * math.pi / 3))


def _cart(a1, a2, f1, f2):
    return f1 * a1[0] + f2 * a2[0], f1 * a1[1] + f2 * a2[1]


def _layers_z(top, nlayers, spacings, jitter, rng):
    z, zs = top, []
    for i in range(nlayers):
        zs.append(z + rng.uniform(-jitter, jitter))
        z -= spacings[i % len(spacings)]
    return zs


def config0_structure(rng, B=0.5, top=-2.0):
    """hex 3.84 A, 4 layers x 2 Si atoms at fractional (0,0), (1/3,2/3),
    layer spacings alternating 0.78 / 2.35 A + U[-0.05, 0.05] jitter."""
    a1, a2 = _hex(3.84)
    zs = _layers_z(top, 4, (0.78, 2.35), 0.05, rng)
    xyz = []
    for z in zs:
        for f1, f2 in ((0.0, 0.0), (1.0 / 3.0, 2.0 / 3.0)):
            x, y = _cart(a1, a2, f1, f2)
            xyz.append((x, y, z))
    n = len(xyz)
    return Structure(np.array(xyz), np.zeros(n, np.int32), np.full(n, B))


def config0():
    rng = np.random.default_rng(1000)
    a1, a2 = _hex(3.84)
    return Workload("cfg0-trhepd-N13-rk4", a1, a2, 13, 10000.0, "positron", -8.0, 400, "rk4",
                    [0.5 + 0.2 * i for i in range(31)], [config0_structure(rng)])


def config1():
    """RHEED: rect 7.68 x 3.84, 8 layers x 4 atoms (Z in {14,32} from seed,
    z-jitter +-0.1), 15 keV electrons, N=61 (mid-shell), 600 slices, sp6,
    121 angles 0.1..6.1 deg."""
    rng = np.random.default_rng(1001)
    a1, a2 = (7.68, 0.0), (0.0, 3.84)
    zs = _layers_z(-1.5, 8, (0.78, 2.35), 0.0, rng)
    xyz, spc, B = [], [], []
    for z in zs:
        for f1, f2 in ((0.0, 0.0), (0.5, 0.0), (0.25, 0.5), (0.75, 0.5)):
            x, y = _cart(a1, a2, f1 + rng.uniform(-0.03, 0.03), f2 + rng.uniform(-0.03, 0.03))
            xyz.append((x, y, z + rng.uniform(-0.1, 0.1)))
            spc.append(int(rng.integers(0, 2)))
            B.append(rng.uniform(0.3, 1.0))
    st = Structure(np.array(xyz), np.array(spc, np.int32), np.array(B))
    return Workload("cfg1-rheed-N61-sp6", a1, a2, 61, 15000.0, "electron", -14.0, 600, "sp6",
                    [0.1 + 0.05 * i for i in range(121)], [st])


def _perturbed_cfg0(rng, n):
    out = []
    for _ in range(n):
        s = config0_structure(rng, B=0.0)
        z = s.xyz[:, 2].copy()
        layers = sorted(set(np.round(z, 12)), reverse=True)[:3]  # top three layers
        for lz in layers:
            dz = rng.uniform(-0.3, 0.3)
            z[np.isclose(z, lz)] += dz
        s.xyz[:, 2] = z
        s.B[:] = rng.uniform(0.3, 1.0)
        out.append(s)
    return out


def config2(n_structures=1024):
    """Global-search batch: 1024 perturbed config-0 structures, N=31, rk4,
    400 slices, 61 angles 0.5..6.5 deg; sharded by structure."""
    rng = np.random.default_rng(1002)
    a1, a2 = _hex(3.84)
    return Workload("cfg2-batch-N31-rk4", a1, a2, 31, 10000.0, "positron", -8.0, 400, "rk4",
                    [0.5 + 0.1 * i for i in range(61)], _perturbed_cfg0(rng, n_structures))


def config3():
    """Many-beam: hex 19.2 A (5x5), 40 atoms / 4 layers seeded, Z in {14,32},
    10 keV positrons, N=199, 1000 slices of 0.01 A, sp6, 61 angles."""
    rng = np.random.default_rng(1003)
    a1, a2 = _hex(19.2)
    zs = _layers_z(-2.0, 4, (0.78, 2.35), 0.05, rng)
    xyz, spc = [], []
    for z in zs:
        for _ in range(10):
            x, y = _cart(a1, a2, rng.uniform(0, 1), rng.uniform(0, 1))
            xyz.append((x, y, z + rng.uniform(-0.1, 0.1)))
            spc.append(int(rng.integers(0, 2)))
    st = Structure(np.array(xyz), np.array(spc, np.int32), np.full(len(xyz), 0.5))
    return Workload("cfg3-manybeam-N199-sp6", a1, a2, 199, 10000.0, "positron", -10.0, 1000, "sp6",
                    [0.5 + 0.1 * i for i in range(61)], [st])


def config4(n_rods=63, method="rk4", n_structures=64, n_angles=64):
    """Throughput sweep: N in {15,31,63,127,255}, config-2 generator,
    64 structures x 64 angles = 4096 pairs, 500 slices, rk4 / sp6."""
    rng = np.random.default_rng(1004)
    a1, a2 = _hex(3.84)
    return Workload(f"cfg4-sweep-N{n_rods}-{method}", a1, a2, n_rods, 10000.0, "positron", -8.0, 500, method,
                    [0.5 + 0.1 * i for i in range(n_angles)], _perturbed_cfg0(rng, n_structures))


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def species_arrays():
    return form_factors()


def product_fields(w):
    """PotentialField objects of the device API for every structure."""
    from . import PotentialField
    ff_a, ff_b = form_factors()
    return [PotentialField.atoms(w.z_bottom, s.xyz, s.species, s.B, ff_a, ff_b, w.cell_area, w.gamma_L, w.sign,
                                 w.absorption, bulk_period=w.bulk_period) for s in w.structures]
