"""Algorithmic work model of one apply/simplify call.

Real flops (2mnk per real GEMM, 8mnk per complex GEMM) in the minimal
contraction order with the materialised, fused-bond target (the reference's
formulation).  F_alg = F_QRpass + F_carry + F_renv + sweeps * F_sweep; the
<T,T> product, the SVDs and the expansions are excluded (as in §8d).
"""
from __future__ import annotations

from typing import Sequence


def qr_pass_bonds(t: Sequence[int], d: Sequence[int]) -> list:
    L = len(d)
    q = [1] * (L + 1)
    for k in range(L - 1):
        q[k + 1] = min(q[k] * d[k], t[k + 1])
    return q


def algorithmic_flops(t: Sequence[int], p: Sequence[int], d: Sequence[int], sweeps: int, complex_: bool = False):
    """t: target bonds (L+1), p: output bonds (L+1), d: physical dims (L)."""
    L = len(d)
    g = 8.0 if complex_ else 2.0  # flops per multiply-add
    q = qr_pass_bonds(t, d)
    f_qr = f_carry = f_renv = f_sweep = 0.0
    for k in range(L - 1):
        m, n = q[k] * d[k], t[k + 1]
        a, b = max(m, n), min(m, n)
        f_qr += (4.0 if complex_ else 1.0) * 4.0 * b * b * (a - b / 3.0)
        f_carry += g * q[k + 1] * t[k + 1] * d[k + 1] * t[k + 2]  # R * T_{k+1}
    for k in range(L - 1, 0, -1):  # truncating R->L: theta V and prev * (U S)
        r = p[k]
        f_carry += g * q[k] * d[k] * p[k + 1] * r + g * q[k - 1] * d[k - 1] * q[k] * r
    for k in range(L - 1, 0, -1):
        f_renv += g * t[k] * d[k] * t[k + 1] * p[k + 1] + g * p[k] * d[k] * p[k + 1] * t[k]
    for n in range(L - 1):
        dn, dn1 = d[n], d[n + 1]
        # left to right: L*T_n, X*T_{n+1}, Y*R^T, env
        f_sweep += g * (p[n] * t[n] * dn * t[n + 1] + p[n] * dn * t[n + 1] * dn1 * t[n + 2]
                        + p[n] * dn * dn1 * t[n + 2] * p[n + 2] + p[n + 1] * p[n] * dn * t[n + 1])
        # right to left: T_{n+1}*R^T, T_n*Z, L*W, env
        f_sweep += g * (t[n + 1] * dn1 * t[n + 2] * p[n + 2] + t[n] * dn * t[n + 1] * dn1 * p[n + 2]
                        + p[n] * t[n] * dn * dn1 * p[n + 2] + p[n + 1] * dn1 * p[n + 2] * t[n + 1])
    total = f_qr + f_carry + f_renv + sweeps * f_sweep
    return dict(F_sweep=f_sweep, F_QRpass=f_qr, F_carry=f_carry, F_renv=f_renv, F_alg=total)
