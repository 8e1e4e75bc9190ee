"""Gauge-invariant comparison of GPU results against the oracle."""
import numpy as np

from oracle import ttlab_oracle as O


def dense(tensors):
    return O.mps_to_dense(O.MPS(tensors))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def spectra(tensors):
    """Per-bond Schmidt spectra from an exact canonical pass (metric 2)."""
    c = O.canonicalize(O.MPS([np.asarray(t) for t in tensors]), 0, O.NO_TRUNCATION)
    out = []
    # move the centre right, recording the singular values of each cut
    psi = O.CanonicalMPS.raw([t.copy() for t in c.tensors], 0)
    for k in range(len(psi) - 1):
        t = psi[k]
        s = O.schmidt_values(t.reshape(-1, t.shape[2]))
        out.append(s)
        psi.move_center_right(O.NO_TRUNCATION)
    return out


def distance(a, b):
    """|a - b| computed cancellation-free: join [a, -b] + exact canonicalization."""
    L = len(a)
    dt = np.result_type(a[0], b[0])
    ts = []
    for n in range(L):
        x, y = a[n].astype(dt), -b[n].astype(dt) if n == 0 else b[n].astype(dt)
        if L == 1:
            ts.append(x + y)
        elif n == 0:
            ts.append(np.concatenate([x, y], axis=2))
        elif n == L - 1:
            ts.append(np.concatenate([x, y], axis=0))
        else:
            t = np.zeros((x.shape[0] + y.shape[0], x.shape[1], x.shape[2] + y.shape[2]), dtype=dt)
            t[:x.shape[0], :, :x.shape[2]] = x
            t[x.shape[0]:, :, x.shape[2]:] = y
            ts.append(t)
    c = O.canonicalize(O.MPS(ts), 0, O.NO_TRUNCATION)
    return c.norm()
