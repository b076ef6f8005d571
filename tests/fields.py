"""Shared test problems: restated from the reference's
proj/tests/support/fields.hpp:17-66 (rect lattice 2.0 x 2.6, 11-rod set,
gamma 2.5, smooth/layered/deep/constant fields) and the closed-form oracles of
proj/tests/support/oracles.hpp:38-49,87-102."""
import cmath
import math

RECT = ((2.0, 0.0), (0.0, 2.6))
K_GAMMA11 = 2.5


def rect_lattice(o):
    return o.Lattice2D(*RECT)


def rods11(o):
    return o.RodSet.build(rect_lattice(o), 5.0)


def rods1(o):
    return o.RodSet.build(rect_lattice(o), 0.5)


# (z_center, amplitude, sigma_xy, sigma_z, absorption)
SMOOTH_LAYERS = [(-5.0, -2.4, 2.2, 80.0, 0.08)]
LAYERED_LAYERS = [(-2.4, -0.22, 2.2, 1.6, 0.08), (-6.0, -0.18, 2.2, 1.9, 0.08)]
DEEP_LAYERS = [(-1.0 - 2.0 * i, -0.22, 2.2, 0.7, 0.08) for i in range(25)]


def smooth_field(o):
    return o.PotentialField.gaussian_layers(-10.0, SMOOTH_LAYERS)


def layered_field(o):
    return o.PotentialField.gaussian_layers(-10.0, LAYERED_LAYERS)


def deep_field(o):
    return o.PotentialField.gaussian_layers(-50.0, DEEP_LAYERS)


def constant_field(o, u, z_e):
    return o.PotentialField.tabulated(z_e, [z_e, 0.0], [((0, 0), [u, u])])


def scalar_gamma(o, gamma, theta0, rods):
    return o.GammaMatrix.build(rods, o.BeamGeometry(gamma, theta0, 0.0))


def fresnel_slab_rho0(g, u, z_e):
    kappa = cmath.sqrt(complex(g * g) + u)
    r = (g - kappa) / (g + kappa)
    E = cmath.exp(2j * kappa * z_e)
    return r * (1.0 - E) / (1.0 - r * r * E)


def fresnel_interface_r(g, u):
    kappa = cmath.sqrt(complex(g * g) + u)
    return (g - kappa) / (g + kappa)


def fit_order(hs, errs, lo=1e-12, hi=1e-3, min_points=3):
    pts = [(math.log(h), math.log(e)) for h, e in zip(hs, errs) if lo < e < hi]
    if len(pts) < min_points:
        return float("nan")
    n = len(pts)
    sx = sum(p[0] for p in pts)
    sy = sum(p[1] for p in pts)
    sxx = sum(p[0] ** 2 for p in pts)
    sxy = sum(p[0] * p[1] for p in pts)
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)
