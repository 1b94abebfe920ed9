"""Post-processing used by the physics checks (reference
pkg/src/sparselbm/validation.py), 3-D: cavity centre-line profiles on the
mid-z plane, Ghia comparison, Poiseuille fit and total mass."""

from dataclasses import dataclass

import numpy as np


@dataclass
class CenterlineProfiles:
    y: np.ndarray
    vx: np.ndarray
    x: np.ndarray
    vy: np.ndarray


def centerline_profiles(simulation, z=None):
    """v_x along the vertical centre line and v_y along the horizontal one on
    the plane z (default mid-plane), normalised by the lid speed
    (reference validation.py:104-126)."""
    if simulation.geometry.provenance.case != "cavity":
        raise ValueError("centerline profiles are defined for the cavity case")
    n_x, n_y, n_z = simulation.geometry.dims
    zc = n_z // 2 if z is None else int(z)
    U = simulation.params.U
    scale = 1.0 / U if U else 1.0
    # two line probes on the device instead of the whole field
    _, vx, _, _ = simulation.macroscopic_box(x=n_x // 2, z=zc)
    _, _, vy, _ = simulation.macroscopic_box(y=n_y // 2, z=zc)
    return CenterlineProfiles(y=np.arange(n_y) / (n_y - 1), vx=vx[0, :, 0] * scale,
                              x=np.arange(n_x) / (n_x - 1), vy=vy[0, 0, :] * scale)


@dataclass
class ProfileComparison:
    mse: float
    max_abs_err: float
    n_samples: int


def compare_to_ghia(profiles, table):
    """Errors against reference samples {"y","u","x","v"} (Ghia 1982), the
    simulated profile linearly interpolated (reference validation.py:137-177)."""
    sq, n, mx = 0.0, 0, 0.0
    for ref_c, ref_v, c, v in ((table["y"], table["u"], profiles.y, profiles.vx),
                               (table["x"], table["v"], profiles.x, profiles.vy)):
        interp = np.interp(ref_c, c, v)
        err = np.abs(interp - ref_v)
        sq += float(np.sum(err ** 2))
        n += err.size
        mx = max(mx, float(err.max()))
    return ProfileComparison(mse=sq / n, max_abs_err=mx, n_samples=n)


@dataclass
class PoiseuilleFit:
    v_max: float
    center: float
    residual: float


def poiseuille_fit(cross_profile, coords=None):
    """Quadratic least squares through a cross-channel profile; returns the
    vertex and 1 - R^2 (reference validation.py:180-206)."""
    v = np.asarray(cross_profile, dtype=np.float64)
    if v.ndim != 1 or v.size < 5:
        raise ValueError("need a 1-D profile with at least 5 samples")
    y = np.arange(v.size, dtype=np.float64) if coords is None else np.asarray(coords, float)
    a, b, c = np.polyfit(y, v, 2)
    ss_tot = float(np.sum((v - v.mean()) ** 2))
    if a >= 0.0 or ss_tot == 0.0:
        return PoiseuilleFit(v_max=float(v.max()), center=float(y[np.argmax(v)]), residual=1.0)
    fitted = a * y * y + b * y + c
    ss_res = float(np.sum((v - fitted) ** 2))
    return PoiseuilleFit(v_max=float(c - b * b / (4.0 * a)), center=float(-b / (2.0 * a)),
                         residual=max(0.0, ss_res / ss_tot))


def total_mass(simulation):
    """Sum of all distribution values over non-solid nodes, float64
    accumulation on the device (reference validation.py:209-215)."""
    return simulation.total_mass()
