"""Config-size parity (SURVEY.md §8c metrics 1-8) for the BASELINE configs whose
CPU oracle takes minutes (C3, C4) and for the batched config C5.

C3/C4 compare the GPU call with oracle results committed under tests/golden/
(`make_config_fixtures.py`: the oracle restatement on the identical seeded
inputs, native dtype).  The oracle's output tensors (`<cfg>_psi_ref.npz`, 6-56 MB)
are git-ignored and travel with the working tree; when present the
cancellation-free distance |psi_gpu - psi_ref| (metric 6) is checked as well.
C5 runs the full 1024-chain batch through the batched engine and compares a
fixed sample of 16 chains with the oracle, run here.
"""
import json
import os

import numpy as np
import pytest

from oracle import ttlab_oracle as O
from paper_2601_16734_b200 import inputs as I

from ._compare import dense, distance, rel, spectra

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


def T():
    from paper_2601_16734_b200 import ttlab
    return ttlab


def _fixture(name):
    with open(os.path.join(GOLDEN, f"{name}_oracle.json")) as f:
        return json.load(f)


def _psi_ref(name):
    p = os.path.join(GOLDEN, f"{name}_psi_ref.npz")
    if not os.path.exists(p):
        return None
    z = np.load(p)
    return [z[f"arr_{i}"] for i in range(len(z.files))]


def _check_against_fixture(name, out, rep, target):
    """Metrics 1-6 and 8 of SURVEY.md §8c against the committed oracle results."""
    t = T()
    fx = _fixture(name)
    tn = np.sqrt(fx["target_norm2"])
    report = {"min_rel_gap_oracle": fx["min_rel_gap"]}
    # 1. output bond dimensions, exact
    assert out.bond_dimensions() == fx["bonds"]
    # 8. sweeps executed
    assert rep["sweeps"] == fx["sweeps"]
    # <T,T> (the engine takes it from the exact QR pass)
    assert abs(rep["target_norm2"] - fx["target_norm2"]) <= 1e-12 * fx["target_norm2"]
    # 3. residual within 1e-10 |T|
    report["residual_abs_diff"] = abs(rep["residual"] - fx["residual"])
    assert report["residual_abs_diff"] <= TOL * tn
    # 4. |psi|
    report["norm_rel"] = abs(rep["norm"] - fx["norm"]) / fx["norm"]
    assert report["norm_rel"] <= TOL
    # 5. <psi, T> (device scalar product against the device target)
    ov = t.scprod(out, target)[0]
    ref_ov = complex(*fx["overlap"])
    report["overlap_rel"] = abs(ov - ref_ov) / abs(ref_ov)
    assert report["overlap_rel"] <= TOL
    ts = out.to_tensors()
    # 2. per-bond Schmidt spectra of the final output (exact canonical pass)
    worst = 0.0
    for s_gpu, s_ref in zip(spectra(ts), fx["spectra"]):
        s_ref = np.asarray(s_ref)
        worst = max(worst, np.linalg.norm(s_gpu - s_ref) / np.linalg.norm(s_ref))
    report["spectra_rel_max"] = worst
    assert worst <= TOL
    # 6. cancellation-free distance to the oracle's output
    ref = _psi_ref(name)
    if ref is not None:
        report["distance_rel"] = distance(ts, ref) / fx["norm"]
        assert report["distance_rel"] <= TOL
    print(name, report)
    return report


def test_config4_full_parity():
    """C4: random D=8 MPO on the n=30, chi=512 MPS, simplify to chi=512 over 2 sweeps
    (simplify.hpp:101-131, mps.hpp:188-218)."""
    t = T()
    cfg = I.CONFIGS["C4"]
    (psi,), W = I.config_inputs(cfg)
    strat = t.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    Wd, pd = t.DeviceMPO(W), t.DeviceMPS.from_tensors(psi)
    rep = []
    out = t.apply(Wd, pd, strat, report=rep)
    target = t.apply_raw(Wd, pd)
    _check_against_fixture("C4", out, rep[0], target)


def test_config3_full_parity():
    """C3: Hadamard product of two complex chi=64 MPS (bond 4096), simplify to chi=128, tol 1e-10."""
    t = T()
    cfg = I.CONFIGS["C3"]
    (a, b), _ = I.config_inputs(cfg)
    strat = t.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    target = t.hadamard(a, b)
    rep = []
    out = t.simplify(target, strat, report=rep)
    _check_against_fixture("C3", out, rep[0], target)


def test_config5_batch_parity():
    """C5: 1024 chains (n=20, chi 128 -> 64) through the batched engine; 16 chains
    (every 64th) against the oracle on metrics 1-4, 7, 8."""
    t = T()
    cfg = I.CONFIGS["C5"]
    chains = I.batch_inputs(cfg, 0, cfg.batch)
    strat = t.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    rep = []
    out = t.simplify(t.DeviceMPS.from_batch(chains), strat, report=rep)
    assert out.count == cfg.batch
    ostrat = O.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    for i in range(0, cfg.batch, 64):
        rr = {}
        ref = O.simplify(O.MPS(chains[i]), ostrat, fast=True, report=rr)
        ts = out.to_tensors(i)
        assert out.bond_dimensions(i) == ref.bond_dimensions()
        assert rep[i]["sweeps"] == rr["sweeps"]
        tn = np.sqrt(rr["target_norm2"])
        assert abs(rep[i]["residual"] - rr["residual"]) <= TOL * tn
        assert abs(rep[i]["norm"] - ref.norm()) <= TOL * ref.norm()
        assert rel(dense(ts), O.mps_to_dense(ref)) <= TOL


def test_config4_repeat_bitwise():
    """Deterministic reductions (split-K partials reduced in fixed order): two C4 calls give
    bitwise identical outputs and reports."""
    t = T()
    cfg = I.CONFIGS["C4"]
    (psi,), W = I.config_inputs(cfg)
    strat = t.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    Wd, pd = t.DeviceMPO(W), t.DeviceMPS.from_tensors(psi)
    r1, r2 = [], []
    a = t.apply(Wd, pd, strat, report=r1).to_tensors()
    b = t.apply(Wd, pd, strat, report=r2).to_tensors()
    assert r1 == r2
    for x, y in zip(a, b):
        assert x.shape == y.shape and np.array_equal(x, y)
