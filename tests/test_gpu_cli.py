"""The B200 CLI (paper_2306_00271_b200/manybeam_b200) driven
by the reference's own CLI suite (proj/tests/test_cli.cpp, built verbatim in
oracle/_ref with MANYBEAM_CLI_PATH pointing at the B200 binary) and by the
reference acceptance gate's criterion 11 (byte determinism across reruns and
--threads 1 vs 8). Plus the extensions: atoms / energy / first-N config keys
give the same curve as the Python API."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2306_00271_b200", "manybeam_b200")


def test_reference_cli_suite_against_b200_cli(ref):
    exe = os.path.join(ROOT, "oracle", "_ref", "tests", "test_cli_b200")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout


def test_acceptance_c11_determinism_with_b200_cli(ref):
    exe = os.path.join(ROOT, "oracle", "_ref", "tests", "acceptance_b200")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    assert len(lines) == 11, r.stdout
    assert all(l.startswith("[PASS]") for l in lines), r.stdout


def workload_json(w, method, dz=None, extra=None):
    """A BASELINE workload as a config document (extension keys)."""
    ff_a, ff_b = configs.form_factors()
    s = w.structures[0]
    cfg = {
        "energy_ev": w.energy_ev, "particle": w.particle,
        "lattice": {"a1": list(w.a1), "a2": list(w.a2)}, "rod_count": w.n_rods,
        "field": {"type": "atoms", "z_bottom": w.z_bottom, "absorption": w.absorption,
                  "species": [{"a": list(a), "b": list(b)} for a, b in zip(ff_a, ff_b)],
                  "atoms": [{"xyz": list(map(float, x)), "species": int(sp), "B": float(B)}
                            for x, sp, B in zip(s.xyz, s.species, s.B)]},
        "angles": {"theta0": list(w.theta0), "theta1": list(w.theta1)},
        "method": method, "slices": w.slices, "dz": dz or -w.z_bottom / w.slices,
    }
    cfg.update(extra or {})
    return cfg


def test_cli_atoms_config_matches_api(tmp_path):
    w = configs.config0().subset(theta0=[0.5, 2.1, 4.7, 6.3])
    p = tmp_path / "c0.json"
    p.write_text(json.dumps(workload_json(w, "rk4")))
    out = tmp_path / "c0.csv"
    r = subprocess.run([CLI, "simulate", "--config", str(p), "--out", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    c = mb.read_curve_csv(str(out))
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    want = mb.rocking_curve(configs.product_fields(w)[0], rods, w.gamma, mb.AngleGrid.validated(w.theta0, w.theta1),
                            mb.SweepOptions(method="rk4", slices=w.slices, dz=-w.z_bottom / w.slices))
    # the CSV carries 15 significant digits
    assert np.abs(np.asarray(c.eta) - want.eta).max() <= 1e-14 * np.abs(want.eta).max() + 1e-300
    # several devices behind one context: byte-identical CSV
    p2 = tmp_path / "c0m.json"
    p2.write_text(json.dumps(workload_json(w, "rk4", extra={"devices": [0, 0]})))
    out2 = tmp_path / "c0m.csv"
    assert subprocess.run([CLI, "simulate", "--config", str(p2), "--out", str(out2)]).returncode == 0
    assert out.read_bytes() == out2.read_bytes()


def test_reference_types_adapter(ref):
    """include/manybeam_b200_ref.hpp: the reference's own PotentialField /
    RodSet / AngleGrid / SweepOptions through manybeam::b200::rocking_curve,
    against manybeam::rocking_curve (oracle/_ref/tests/adapter_b200)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "tests", "adapter_b200")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed" in r.stdout
