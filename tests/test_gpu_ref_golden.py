"""CUDA path vs outputs of the REFERENCE'S OWN CODE (tests/golden/ref_outputs.npz, produced by
oracle/_ref/ttlab_ref; see tests/ref_cases.py).  No oracle in between: the inputs are regenerated
from seeds, pushed through the C-ABI and compared with the reference outputs on the
gauge-invariant results (bond dimensions, sweeps, error ledger, norm, distance <= 1e-10)."""
import numpy as np
import pytest

from . import ref_cases as R
from .test_oracle_vs_ref import FIX, check_against_reference

pytestmark = pytest.mark.gpu


def run_gpu(name):
    from paper_2601_16734_b200 import ttlab as t
    op, st, inp = R.case(name)
    s = t.Strategy(method=st["method"], tolerance=st["tolerance"],
                   simplification_tolerance=st["simplification_tolerance"],
                   max_bond=st["max_bond"] or t.UNBOUNDED_BOND, max_sweeps=st["max_sweeps"],
                   normalize=st["normalize"])
    rep = []
    if op == "apply":
        out = t.apply(inp["mpo"], inp["mps"][0], s, report=rep)
    elif op == "hadamard_simplify":
        out = t.simplify(t.hadamard(inp["mps"][0], inp["mps"][1]), s, report=rep)
    elif op == "simplify":
        out = t.simplify(inp["mps"][0], s, inp.get("guess"), report=rep)
    elif op == "canonicalize":
        out = t.canonicalize(inp["mps"][0], inp["center"], s, report=rep)
    elif op == "simplify_sum":
        out = t.simplify(t.MPSSum(inp["weights"], inp["mps"]), s, report=rep)
    elif op == "apply_sum":
        out = t.apply(inp["mpo"], t.MPSSum(inp["weights"], inp["mps"]), s, report=rep)
    elif op in ("qft", "iqft"):
        from paper_2601_16734_b200 import qft as Q
        out = (Q.qft if op == "qft" else Q.iqft)(inp["mps"][0], s)
    elif op == "heff":
        # operator environments on the device (ttg_op_env_update, device buffers) + the device matvec
        import ctypes as C
        import torch
        from paper_2601_16734_b200 import _lib
        W, bra, ket, k = inp["mpo"], inp["mps"][0], inp["mps"][1], inp["site"]
        _, _, x = R.heff_inputs(W, bra, ket, k)
        ctx = t.context()

        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.complex128)).cuda()

        def step(env, i, side):
            b, w, kt = np.asarray(bra[i]), np.asarray(W[i]), np.asarray(ket[i])
            Dl, dout, din, Dr = w.shape
            dims = (C.c_int * 8)(Dl, dout, din, Dr, b.shape[0], b.shape[2], kt.shape[0], kt.shape[2])
            shape = (Dr, b.shape[2], kt.shape[2]) if side == 0 else (Dl, b.shape[0], kt.shape[0])
            out = torch.empty(shape, dtype=torch.complex128, device="cuda")
            bufs = [env, dev(b), dev(w), dev(kt)]
            torch.cuda.synchronize()
            ctx.check(_lib.lib.ttg_op_env_update(ctx.handle, _lib.TTG_C128, side, dims,
                                                 *[C.c_void_p(z.data_ptr()) for z in bufs], C.c_void_p(out.data_ptr())))
            ctx.synchronize()
            return out

        L = dev(np.ones((1, 1, 1)))
        for i in range(k):
            L = step(L, i, 0)
        Rr = dev(np.ones((1, 1, 1)))
        for i in range(len(ket) - 1, k + 1, -1):
            Rr = step(Rr, i, 1)
        y = t.apply_effective_two_site(L.cpu().numpy(), np.asarray(W[k], dtype=np.complex128),
                                       np.asarray(W[k + 1], dtype=np.complex128), Rr.cpu().numpy(), x)
        return {"size": int(np.asarray(y).size)}, [np.asarray(y).reshape(1, -1, 1)]
    elif op == "scprod":
        v = complex(t.scprod(inp["mps"][0], inp["mps"][1])[0])
        return {"re": v.real, "im": v.imag}, None
    elif op == "expectation_mpo":
        v = complex(t.expectation_mpo(inp["mpo"], inp["mps"][0], inp["mps"][1])[0])
        return {"re": v.real, "im": v.imag}, None
    else:
        raise ValueError(op)
    ts = out.to_tensors()
    meta = {"error": float(out.error()), "norm": float(t.norm(out)[0]), "bonds": [int(x.shape[2]) for x in ts]}
    if rep and st["method"] == R.V and op in ("simplify", "apply", "hadamard_simplify"):
        meta["sweeps"] = int(rep[0]["sweeps"])
    return meta, ts


@pytest.mark.parametrize("name", list(R.CASES))
def test_gpu_matches_reference_output(name):
    ref_meta, ref_tensors = FIX[name]
    meta, tensors = run_gpu(name)
    if "sweeps" not in ref_meta:
        meta.pop("sweeps", None)
    check_against_reference(name, meta, tensors, ref_meta, ref_tensors)
