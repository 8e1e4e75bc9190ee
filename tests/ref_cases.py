"""Cases run through the REFERENCE ITSELF (oracle/_ref/ttlab_ref: the reference's own headers
compiled against the Eigen stand-in, oracle/Makefile) to pin the oracle and the CUDA path.

TEST INFRASTRUCTURE.  One table, three consumers:
  tests/golden/make_ref_fixtures.py  runs every case through ttlab_ref and commits the outputs;
  tests/test_oracle_vs_ref.py        (CPU) oracle restatement vs those reference outputs;
  tests/test_gpu_ref_golden.py       (GPU) CUDA path vs the same reference outputs.
Inputs are regenerated from seeds (bit-exact generators), so only outputs are stored.
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile

import numpy as np

from oracle import ttlab_oracle as O
from oracle.rng import random_matrix
from paper_2601_16734_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ttlab_ref")
FIXTURE = os.path.join(ROOT, "tests", "golden", "ref_outputs.npz")

S, V = 0, 1  # Truncation::SVD_TRUNCATE, VARIATIONAL (types.hpp:39)


def strat(method=V, tolerance=1e-12, simplification_tolerance=1e-12, max_bond=0, max_sweeps=4, normalize=False):
    return dict(method=method, tolerance=tolerance, simplification_tolerance=simplification_tolerance,
                max_bond=max_bond, max_sweeps=max_sweeps, normalize=normalize)


def _ru(L, d, bond, seed):
    return O.random_uniform_mps(L, d, bond, seed).tensors


def _rank_deficient(L, seed):
    """hadamard(u, u): bonds 9 with Schmidt rank <= 6 (symmetric square of a bond-3 state)."""
    u = O.random_uniform_mps(L, 2, 3, seed)
    return O.hadamard(u, u).tensors


def _local_mpo_sum(L, seeds_a, seeds_b):
    a = O.mpo_from_local_operators([random_matrix(2, 2, s) for s in seeds_a])
    b = O.mpo_from_local_operators([random_matrix(2, 2, s) for s in seeds_b])
    return O.mpo_sum([0.5 + 0.25j, -1 + 1j], [a, b]).tensors


def _cfg(name):
    cfg = I.CONFIGS[name]
    mps, W = I.config_inputs(cfg)
    return cfg, mps, W


def _cfg_strat(cfg):
    return strat(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)


# name -> (op, strategy, inputs builder).  inputs: dict(mps=[...], mpo=..., weights=[...], center=int, guess=...)
CASES = {
    # --- simplify (simplify.hpp:182-195)
    "simplify_uniform_n10_chi16_to6": ("simplify", strat(max_bond=6), lambda: dict(mps=[_ru(10, 2, 16, 7)])),
    "simplify_normal_n12_chi32_to12": ("simplify", strat(max_bond=12),
                                       lambda: dict(mps=[I.random_mps(12, 2, 32, 500)])),
    "simplify_complex_n10_tol1e-6": ("simplify", strat(tolerance=1e-6, max_sweeps=6),
                                     lambda: dict(mps=[I.random_mps(10, 2, 16, 11, complex_=True)])),
    "simplify_normalize_n9_d3": ("simplify", strat(max_bond=5, normalize=True), lambda: dict(mps=[_ru(9, 3, 9, 13)])),
    "simplify_svd_method_n10": ("simplify", strat(method=S, max_bond=7), lambda: dict(mps=[_ru(10, 2, 16, 17)])),
    "simplify_with_guess_n10": ("simplify", strat(max_bond=6, max_sweeps=3),
                                lambda: dict(mps=[_ru(10, 2, 16, 7)], guess=_ru(10, 2, 4, 8))),
    "simplify_two_sites": ("simplify", strat(max_bond=1), lambda: dict(mps=[_ru(2, 2, 2, 3)])),
    "simplify_one_site": ("simplify", strat(), lambda: dict(mps=[_ru(1, 3, 1, 4)])),
    "simplify_product_state": ("simplify", strat(max_bond=4), lambda: dict(mps=[_ru(8, 2, 1, 5)])),
    "simplify_config_C1": ("simplify", None, lambda: dict(mps=[_cfg("C1")[1][0]])),
    "simplify_chain0_config_C5": ("simplify", None, lambda: dict(mps=[I.config_inputs(I.CONFIGS["C5"], chain=0)[0][0]])),
    # --- canonicalize (mps.hpp:188-218, 310-313)
    "canonicalize_c0_chi5": ("canonicalize", strat(method=S, max_bond=5), lambda: dict(mps=[_ru(10, 2, 16, 7)], center=0)),
    "canonicalize_c3_chi5": ("canonicalize", strat(method=S, max_bond=5), lambda: dict(mps=[_ru(10, 2, 16, 7)], center=3)),
    "canonicalize_c9_tol1e-3": ("canonicalize", strat(method=S, tolerance=1e-3),
                                lambda: dict(mps=[_ru(10, 2, 16, 19)], center=9)),
    "canonicalize_exact_rank_deficient": ("canonicalize", strat(method=S, tolerance=0.0, simplification_tolerance=0.0),
                                          lambda: dict(mps=[_rank_deficient(8, 23)], center=2)),
    "canonicalize_default_rank_deficient": ("canonicalize", strat(method=S),
                                            lambda: dict(mps=[_rank_deficient(8, 23)], center=0)),
    # --- apply (blas.hpp:8-11)
    "apply_laplacian_n12_chi16": ("apply", strat(max_bond=16), lambda: dict(mpo=I.laplacian_mpo(12),
                                                                            mps=[I.random_mps(12, 2, 16, 202)])),
    "apply_random_D4_n10_chi8": ("apply", strat(max_bond=8, max_sweeps=2),
                                 lambda: dict(mpo=I.random_mpo(10, 2, 4, 406), mps=[I.random_mps(10, 2, 8, 405)])),
    "apply_complex_local_sum_n4": ("apply", strat(), lambda: dict(mpo=_local_mpo_sum(4, (1, 2, 3, 4), (5, 6, 7, 8)),
                                                                  mps=[_ru(4, 2, 3, 31)])),
    "apply_random_D8_n14_chi32": ("apply", strat(max_bond=32, max_sweeps=2),
                                  lambda: dict(mpo=I.random_mpo(14, 2, 8, 406), mps=[I.random_mps(14, 2, 32, 405)])),
    "apply_config_C2": ("apply", None, lambda: dict(mpo=_cfg("C2")[2], mps=[_cfg("C2")[1][0]])),
    # --- hadamard + simplify (blas.hpp:45-67)
    "hadamard_complex_n10_chi6": ("hadamard_simplify", strat(max_bond=12, tolerance=1e-10),
                                  lambda: dict(mps=[I.random_mps(10, 2, 6, 303, complex_=True),
                                                    I.random_mps(10, 2, 6, 304, complex_=True)])),
    "hadamard_complex_n12_chi16": ("hadamard_simplify", strat(max_bond=32, tolerance=1e-10),
                                   lambda: dict(mps=[I.random_mps(12, 2, 16, 303, complex_=True),
                                                     I.random_mps(12, 2, 16, 304, complex_=True)])),
    # --- sums (simplify.hpp:198-215, blas.hpp:13-20)
    "simplify_sum_3terms": ("simplify_sum", strat(max_bond=8),
                            lambda: dict(mps=[_ru(8, 2, 4, 41), _ru(8, 2, 6, 42), _ru(8, 2, 3, 43)],
                                         weights=[0.5 + 0.25j, -1.0 + 0j, 0.3 - 0.7j])),
    "simplify_sum_svd_method": ("simplify_sum", strat(method=S, max_bond=6),
                                lambda: dict(mps=[_ru(8, 2, 4, 41), _ru(8, 2, 6, 42)], weights=[1.0 + 0j, -0.5 + 0j])),
    "apply_sum_2terms": ("apply_sum", strat(max_bond=8),
                         lambda: dict(mpo=I.laplacian_mpo(8), mps=[I.random_mps(8, 2, 4, 51), I.random_mps(8, 2, 6, 52)],
                                      weights=[1.0 + 0j, 2.0 + 0j])),
    # --- MPO lists: the Fourier transform circuit (qft.hpp:68-113 through apply(MPOList), blas.hpp:24-32)
    "qft_uniform_n8": ("qft", strat(), lambda: dict(mps=[_ru(8, 2, 4, 71)])),
    "iqft_complex_n10_chi8": ("iqft", strat(max_bond=8), lambda: dict(mps=[I.random_mps(10, 2, 8, 72, complex_=True)])),
    "qft_product_state_n12": ("qft", strat(tolerance=1e-10), lambda: dict(mps=[_ru(12, 2, 1, 73)])),
    # --- operator environments + two-site effective operator matvec (environments.hpp:42-83, eigensolvers.hpp:15-64)
    "heff_laplacian_n8_site3": ("heff", strat(), lambda: dict(mpo=I.laplacian_mpo(8), site=3,
                                                              mps=[I.random_mps(8, 2, 6, 81, complex_=True)] * 2)),
    "heff_random_D4_bra_ne_ket": ("heff", strat(), lambda: dict(mpo=I.random_mpo(8, 2, 4, 82), site=2,
                                                                mps=[I.random_mps(8, 2, 5, 83), I.random_mps(8, 2, 7, 84)])),
    # --- scalars (mps.hpp:416-423, blas.hpp:128-138)
    "scprod_uniform": ("scprod", strat(), lambda: dict(mps=[_ru(9, 2, 5, 61), _ru(9, 2, 7, 62)])),
    "expectation_local_sum": ("expectation_mpo", strat(),
                              lambda: dict(mpo=_local_mpo_sum(4, (51, 52, 53, 54), (55, 56, 57, 58)),
                                           mps=[_ru(4, 2, 2, 17), _ru(4, 2, 3, 18)])),
    "expectation_laplacian_n12": ("expectation_mpo", strat(),
                                  lambda: dict(mpo=I.laplacian_mpo(12), mps=[I.random_mps(12, 2, 16, 7)] * 2)),
}


def case(name):
    op, st, build = CASES[name]
    inp = build()
    if st is None:  # BASELINE config
        cfg = I.CONFIGS[name.rsplit("_", 1)[1]]
        st = _cfg_strat(cfg)
    return op, st, inp


def ostrategy(st):
    return O.Strategy(method=st["method"], tolerance=st["tolerance"],
                      simplification_tolerance=st["simplification_tolerance"],
                      max_bond=st["max_bond"] or O.UNBOUNDED_BOND, max_sweeps=st["max_sweeps"],
                      normalize=st["normalize"])


def _omps(ts):
    return O.MPS([np.asarray(t) for t in ts], 0.0)


# ----------------------------------------------------------------------------- reference runs
def _strategy_arg(st):
    return "%s:%r:%r:%d:%d:%d" % ("S" if st["method"] == S else "V", float(st["tolerance"]),
                                  float(st["simplification_tolerance"]), int(st["max_bond"]),
                                  int(st["max_sweeps"]), int(st["normalize"]))


def have_ref():
    return os.path.exists(REF_BIN)


def run_reference(name, timeout=3600):
    """Run one case through oracle/_ref/ttlab_ref.  Returns (meta dict, output tensors or None)."""
    op, st, inp = case(name)
    with tempfile.TemporaryDirectory() as tmp:
        def put_mps(i, ts):
            p = os.path.join(tmp, "s%d.ttlab" % i)
            with open(p, "wb") as f:
                f.write(O.dumps_mps(_omps(ts)))
            return p

        args = []
        if "mpo" in inp and op in ("apply", "apply_sum", "expectation_mpo", "heff"):
            p = os.path.join(tmp, "w.ttlab")
            with open(p, "wb") as f:
                f.write(O.dumps_mpo(O.MPO([np.asarray(t) for t in inp["mpo"]])))
            args.append(p)
        files = [put_mps(i, ts) for i, ts in enumerate(inp["mps"])]
        if op in ("simplify_sum", "apply_sum"):
            args.append(str(len(files)))
            for w, p in zip(inp["weights"], files):
                args += [repr(float(np.real(w))), repr(float(np.imag(w))), p]
        elif op == "canonicalize":
            args = [str(inp["center"])] + files
        elif op == "heff":
            args += files + [str(inp["site"])]
        else:
            args += files
        if inp.get("guess") is not None:
            args.append(put_mps(99, inp["guess"]))
        outp = os.path.join(tmp, "out.ttlab")
        r = subprocess.run([REF_BIN, op, outp, _strategy_arg(st)] + args, capture_output=True, text=True,
                           timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError("ttlab_ref %s failed (%d): %s %s" % (name, r.returncode, r.stdout, r.stderr))
        meta = json.loads(r.stdout.strip().splitlines()[-1])
        tensors = None
        if op == "heff":  # raw complex128 vector y = H_eff x, stored as one (1, size, 1) "site"
            y = np.fromfile(outp, dtype=np.complex128)
            assert y.size == meta["size"] and meta["dense_diff"] <= 1e-12 * max(meta["ynorm"], 1.0)
            return meta, [y.reshape(1, -1, 1)]
        if os.path.exists(outp):
            with open(outp, "rb") as f:
                out = O.loads_mps(f.read())
            tensors = out.tensors
            assert abs(out.error - meta["error"]) <= 1e-15 * max(1.0, abs(meta["error"]))
    return meta, tensors


# ----------------------------------------------------------------------------- fixtures
def load_fixture():
    z = np.load(FIXTURE, allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    out = {}
    for name, m in meta.items():
        ts = None
        if m.get("sites") is not None:
            ts = []
            for k in range(m["sites"]):
                t = z["%s/%d" % (name, k)]
                ts.append(t)
        out[name] = (m, ts)
    return out


def heff_inputs(W, bra, ket, k):
    """Oracle operator environments around the pair (k, k+1) and x = join_pair(ket pair), complex128."""
    n = len(ket)
    L = np.ones((1, 1, 1), dtype=np.complex128)
    for i in range(k):
        L = O.update_left_op_environment(L, np.asarray(bra[i]), np.asarray(W[i]), np.asarray(ket[i]))
    R = np.ones((1, 1, 1), dtype=np.complex128)
    for i in range(n - 1, k + 1, -1):
        R = O.update_right_op_environment(R, np.asarray(bra[i]), np.asarray(W[i]), np.asarray(ket[i]))
    x = np.einsum("asb,btc->astc", np.asarray(ket[k]), np.asarray(ket[k + 1])).reshape(-1).astype(np.complex128)
    return L, R, x


def _qft_layers_host(L, inverse):
    """The circuit layers as host tensors (paper_2601_16734_b200/qft.py builds them on the host; they are
    checked against the oracle's dense circuit in tests/test_qft_host.py)."""
    from paper_2601_16734_b200 import qft as Q
    sign = 1.0 if inverse else -1.0
    order = range(L) if inverse else range(L - 1, -1, -1)  # qft.hpp:84-100: matrix order, last factor acts first
    return [Q.qft_layer(L, list(range(L)), m, sign, inverse) for m in order]


# ----------------------------------------------------------------------------- oracle runs
def run_oracle(name):
    """The oracle restatement on the same case: (meta, tensors)."""
    op, st, inp = case(name)
    s = ostrategy(st)
    rep = {}
    if op == "apply":
        out = O.apply(O.MPO(inp["mpo"]), _omps(inp["mps"][0]), s, report=rep)
    elif op == "hadamard_simplify":
        out = O.simplify(O.hadamard(_omps(inp["mps"][0]), _omps(inp["mps"][1])), s, report=rep)
    elif op == "simplify":
        g = inp.get("guess")
        out = O.simplify(_omps(inp["mps"][0]), s, None if g is None else _omps(g), report=rep)
    elif op == "canonicalize":
        out = O.canonicalize(_omps(inp["mps"][0]), inp["center"], s)
    elif op == "simplify_sum":
        out = O.simplify_sum(O.MPSSum(inp["weights"], [_omps(t) for t in inp["mps"]]), s)
    elif op == "apply_sum":
        out = O.apply_sum(O.MPO(inp["mpo"]), O.MPSSum(inp["weights"], [_omps(t) for t in inp["mps"]]), s)
    elif op in ("qft", "iqft"):
        layers = _qft_layers_host(len(inp["mps"][0]), op == "iqft")
        out = _omps(inp["mps"][0])
        for layer in reversed(layers):  # the last factor acts first (blas.hpp:24-32)
            out = O.apply(O.MPO(layer), out, s)
    elif op == "heff":
        W, bra, ket, k = inp["mpo"], inp["mps"][0], inp["mps"][1], inp["site"]
        L, R, x = heff_inputs(W, bra, ket, k)
        y = O.apply_effective_two_site(L, np.asarray(W[k]), np.asarray(W[k + 1]), R, x)
        return {"size": int(y.size), "ynorm": float(np.linalg.norm(y))}, [np.asarray(y).reshape(1, -1, 1)]
    elif op == "scprod":
        v = O.scprod(_omps(inp["mps"][0]), _omps(inp["mps"][1]))
        return {"re": float(np.real(v)), "im": float(np.imag(v))}, None
    elif op == "expectation_mpo":
        v = O.expectation_mpo(O.MPO(inp["mpo"]), _omps(inp["mps"][0]), _omps(inp["mps"][1]))
        return {"re": float(np.real(v)), "im": float(np.imag(v))}, None
    else:
        raise ValueError(op)
    meta = {"error": float(out.error), "norm": float(out.norm()), "bonds": [int(t.shape[2]) for t in out.tensors]}
    if "sweeps" in rep:
        meta["sweeps"] = int(rep["sweeps"])
        meta["residual"] = float(rep["residual"])
    if hasattr(out, "center"):
        meta["center"] = int(out.center)
    return meta, out.tensors
