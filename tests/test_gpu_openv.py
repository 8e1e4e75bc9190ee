"""Device operator environments and the device-pointer two-site effective operator against the
oracle (environments.hpp:42-83, eigensolvers.hpp:15-64)."""
import ctypes as C

import numpy as np
import pytest

from oracle import ttlab_oracle as O

pytestmark = pytest.mark.gpu


def _ctx():
    from paper_2601_16734_b200 import ttlab
    return ttlab.context()


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("complex_", [False, True])
@pytest.mark.parametrize("side", [0, 1])
def test_op_env_update_matches_oracle(complex_, side):
    import torch
    from paper_2601_16734_b200 import _lib
    rng = np.random.default_rng(7 + side)
    Dl, dout, din, Dr, al, ar, bl, br = 3, 2, 2, 4, 5, 6, 7, 3

    def rnd(*s):
        x = rng.standard_normal(s)
        return x + 1j * rng.standard_normal(s) if complex_ else x

    bra, op, ket = rnd(al, dout, ar), rnd(Dl, dout, din, Dr), rnd(bl, din, br)
    if side == 0:
        env = rnd(Dl, al, bl)
        ref = O.update_left_op_environment(env, bra, op, ket)
        out = torch.empty((Dr, ar, br), dtype=torch.complex128 if complex_ else torch.float64, device="cuda")
    else:
        env = rnd(Dr, ar, br)
        ref = O.update_right_op_environment(env, bra, op, ket)
        out = torch.empty((Dl, al, bl), dtype=torch.complex128 if complex_ else torch.float64, device="cuda")
    ctx = _ctx()
    dims = (C.c_int * 8)(Dl, dout, din, Dr, al, ar, bl, br)
    t = [_dev(x) for x in (env, bra, op, ket)]
    torch.cuda.synchronize()
    ctx.check(_lib.lib.ttg_op_env_update(ctx.handle, _lib.TTG_C128 if complex_ else _lib.TTG_F64, side, dims,
                                         *[C.c_void_p(x.data_ptr()) for x in t], C.c_void_p(out.data_ptr())))
    ctx.synchronize()
    got = out.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_heff_device_matches_host_variant():
    """ttg_apply_effective_two_site_dev (device buffers, no host copies) equals the host variant and
    <psi|H|psi> through the device operator environments."""
    import torch
    from paper_2601_16734_b200 import _lib, ttlab
    rng = np.random.default_rng(3)
    D0, D1, D2, d = 4, 8, 4, 2
    chiA, chiB = 24, 20
    L = rng.standard_normal((D0, chiA, chiA))
    R = rng.standard_normal((D2, chiB, chiB))
    w1 = rng.standard_normal((D0, d, d, D1))
    w2 = rng.standard_normal((D1, d, d, D2))
    x = rng.standard_normal((chiA, d, d, chiB))
    y_host = ttlab.apply_effective_two_site(L, w1, w2, R, x)
    ctx = _ctx()
    dims = (C.c_int * 11)(D0, D1, D2, d, d, d, d, chiA, chiA, chiB, chiB)
    t = [_dev(a) for a in (L, w1, w2, R, x)]
    y = torch.empty(y_host.shape, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.check(_lib.lib.ttg_apply_effective_two_site_dev(ctx.handle, _lib.TTG_F64, dims,
                                                        *[C.c_void_p(a.data_ptr()) for a in t],
                                                        C.c_void_p(y.data_ptr())))
    ctx.synchronize()
    assert np.abs(y.cpu().numpy().reshape(y_host.shape) - y_host).max() <= 1e-12 * np.abs(y_host).max()
    ref = O.apply_effective_two_site(L, w1, w2, R, x)
    assert np.abs(y.cpu().numpy().reshape(ref.shape) - ref).max() <= 1e-12 * np.abs(ref).max()
